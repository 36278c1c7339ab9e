"""Multi-process (world_size 2, gloo, CPU) test of the chunk-shard plan of
nc_compress_shard: each rank owns a contiguous chunk range,
the only exchange is an allgather of the 12-byte chunk-table entries, and each
rank emits its byte range of the final NC05 container.  The per-chunk streams
come from the CPU oracle (no GPU here); the plan, the gathered table and the
part assembly run through libnc's host functions.  Concatenating the parts
must equal the single-process container (worker independence)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2602_19626_b200 as nc
    from oracle.ensemble import Params, encode_tokens
    from oracle.lm import LM
    from oracle.ncw import Weights
    from oracle.tokenizer import Tokenizer
    from synth import ensure_model, make_text

    w = Weights(ensure_model("tiny"))
    data = make_text("alice", 2500, 31)
    n_chunks = 5
    prm = Params(window=16, slide=4, warmup=10, n_chunks=n_chunks)
    cuts = nc.nc_host_split(data, n_chunks)
    nch = len(cuts) - 1
    c0, c1 = nc.nc_host_shard_range(nch, world, rank)
    k = -(-nch // world)
    tk, lm = Tokenizer(w.vocab), LM(w)
    mine, streams = [], b""
    for c in range(c0, c1):
        t = tk.encode(data[cuts[c]:cuts[c + 1]])
        x = [w.bos] + t[:-1] if t else []
        r = encode_tokens(lm.forward_blocked(x, prm.window, prm.slide), t, w.V, prm)
        mine += [len(t), r["bits"], len(r["stream"])]
        streams += r["stream"]
    mine += [0] * (3 * k - len(mine))
    gathered = [torch.zeros(3 * k, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(gathered, torch.tensor(mine, dtype=torch.int64))
    table = np.concatenate([g.numpy() for g in gathered]).reshape(-1, 3)[:nch]
    part, off, total = nc.nc_host_shard_part(table.astype(np.uint32), prm.flags, prm.tau_milli, world, rank, streams)
    parts = [None] * world
    dist.all_gather_object(parts, (off, part, total))
    if rank == 0:
        with open(os.path.join(out_dir, "parts.bin"), "wb") as f:
            import pickle
            pickle.dump(parts, f)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shard_plan(tmp_path, tiny_weights):
    import pickle

    import __graft_entry__
    __graft_entry__.build()
    from oracle.compressor import compress
    from oracle.ensemble import Params
    from synth import make_text
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    parts = pickle.load(open(tmp_path / "parts.bin", "rb"))
    parts.sort(key=lambda x: x[0])
    total = parts[0][2]
    blob = b"".join(p for _, p, _ in parts)
    assert all(t == total for _, _, t in parts) and len(blob) == total
    assert parts[1][0] == len(parts[0][1])          # contiguous byte ranges
    ref = compress(make_text("alice", 2500, 31), tiny_weights,
                   Params(window=16, slide=4, warmup=10, n_chunks=5))
    assert blob == ref


def _dec_worker(rank, world, port, out_dir, blob):
    """Decompress side of the shard plan: every rank parses the full
    container, decodes its chunk range, and one allgather of decoded byte lengths gives
    its output offset (as nc_decompress_shard does over NCCL)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import pickle

    import paper_2602_19626_b200 as nc
    from oracle.container import read_nc05
    from oracle.ensemble import Params, decode_tokens
    from oracle.lm import LM
    from oracle.ncw import Weights
    from oracle.tokenizer import Tokenizer
    from synth import ensure_model

    w = Weights(ensure_model("tiny"))
    flags, tau_milli, chunks = read_nc05(blob)
    prm = Params(window=16, slide=4, warmup=10, n_chunks=len(chunks), flags=flags)
    c0, c1 = nc.nc_host_shard_range(len(chunks), world, rank)
    tk, lm = Tokenizer(w.vocab, w.n_special), LM(w)
    text = b""
    for n, bits, stream in chunks[c0:c1]:
        inc = lm.incremental(prm.window, prm.slide)
        toks = decode_tokens(lambda x, inc=inc: inc.step(w.bos if x is None else x), n, stream, w.V, prm)
        text += tk.decode(toks)
    lens = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(lens, torch.tensor([len(text)], dtype=torch.int64))
    off = int(sum(int(l) for l in lens[:rank]))
    tot = int(sum(int(l) for l in lens))
    with open(os.path.join(out_dir, f"dec{rank}.bin"), "wb") as f:
        pickle.dump((off, text, tot, c1 - c0), f)
    dist.barrier()
    dist.destroy_process_group()


def test_three_rank_decompress_plan(tmp_path, tiny_weights):
    """4 chunks over 3 ranks (2, 2, 0 chunks: one rank decodes nothing); the parts,
    placed at their gathered offsets, rebuild the input exactly."""
    import pickle

    import __graft_entry__
    __graft_entry__.build()
    from oracle.compressor import compress
    from oracle.ensemble import Params
    from synth import make_text
    data = make_text("alice", 2000, 37)
    blob = compress(data, tiny_weights, Params(window=16, slide=4, warmup=10, n_chunks=4))
    mp.spawn(_dec_worker, args=(3, _free_port(), str(tmp_path), blob), nprocs=3, join=True)
    parts = [pickle.load(open(tmp_path / f"dec{r}.bin", "rb")) for r in range(3)]
    assert [p[3] for p in parts] == [2, 2, 0]
    assert all(p[2] == len(data) for p in parts)
    out = bytearray(len(data))
    for off, text, _, _ in parts:
        out[off:off + len(text)] = text
    assert bytes(out) == data
    assert parts[1][0] == len(parts[0][1]) and parts[2][0] == len(data)
