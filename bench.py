#!/usr/bin/env python
"""Benchmark: compress bytes/s of the Nacrith hot path on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload config3]

One step = one full compression of the workload (SURVEY.md §8(a) rows a1-a10:
embed, 30 x {RMSNorm+QKV+RoPE, window attention, O, RMSNorm+SwiGLU MLP},
head, the per-token CDF walk, host range coding, NC05 assembly).

Workloads (synth/configs.py, BASELINE.json configs): the default is config3 -- the
metric's "1/2/4/8 B200" workload: 10 MB alice-shaped text, 64 chunks per GPU,
STRONG scaling (the same 10 MB at every N, 64 N chunks: SURVEY §8(d)/(e)).
config4_shard (12.5 MB enwik-shaped per GPU, 64 chunks per GPU) and config2
(152 KB, 8 chunks per GPU) scale weakly (each rank owns its own copy-sized share).

value : device-resident inputs (token ids already in HBM) -> NC05 container
        through nc_compress_tokens; CUDA events on the launching stream,
        barrier + synchronize around every step, max over ranks.
e2e   : the same through nc_compress / nc_compress_shard (host bytes in,
        container out: tokenization, H2D of the token ids, D2H of the (cum, freq)
        pairs, the NCCL allgather of the chunk table for N > 1).
--gpus N without a torchrun environment re-launches itself under
torch.distributed.run with N ranks (one per GPU, NCCL); rank 0 prints the line.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "sm_max_mhz": 1965.0}
N_SM = 148


def peaks():
    try:
        with open(PEAKS_FILE) as f:
            return json.load(f), "measured"
    except Exception:
        return FALLBACK, "fallback"


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, device):
        self.device, self.proc, self.path = device, None, None

    def start(self):
        try:
            os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
            self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=index,clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 9 and f[1].isdigit():
                rows.append(f)
        if not rows:
            return None
        sm = [int(r[1]) for r in rows]
        load = [int(r[1]) for r in rows if float(r[3] or 0) > 200] or sm
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for n, v in zip(names, r[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": int(statistics.median(load)), "sm_max_mhz": int(rows[0][2]), "reasons": sorted(reasons),
                "samples": len(rows)}


# ------------------------------------------------------------------ oracle ---
def _oracle_worker(job):
    """one chunk's sample through the CPU oracle (as it stands): blocked fp64 forward +
    ensemble walk + WNC on the first n tokens of the chunk.  Runs in a pool process."""
    path, chunk, n_tokens, window, slide, cdf_bits, blas = job
    from threadpoolctl import threadpool_limits
    threadpool_limits(blas)          # the pool was forked after numpy loaded its BLAS
    from oracle.ensemble import Params, encode_tokens
    from oracle.lm import LM
    from oracle.ncw import Weights
    from oracle.tokenizer import Tokenizer
    w = _oracle_worker.cache.get(path)
    if w is None:
        w = _oracle_worker.cache[path] = Weights(path)
    tk = Tokenizer(w.vocab)
    t = tk.encode(chunk)[:n_tokens]
    prm = Params(window=window, slide=slide, cdf_bits=cdf_bits)
    t0 = time.perf_counter()
    Z = LM(w).forward_blocked([w.bos] + t[:-1], prm.window, prm.slide)
    encode_tokens(Z, t, w.V, prm)
    return len(tk.decode(t)), len(t), time.perf_counter() - t0


_oracle_worker.cache = {}


class OraclePool:
    """SURVEY §8(d) oracle timing: chunk-parallel multiprocessing, P = min(8, cores) workers
    (one chunk each, the first P chunks of the workload), BLAS threads = cores / P."""

    def __init__(self, path, data, wl, n_chunks):
        import multiprocessing as mp
        from oracle.chunking import split_chunks
        cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
        self.P = max(1, min(8, cores, n_chunks))
        self.blas = max(1, cores // self.P)
        self.cores = self.P * self.blas
        for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
            os.environ[k] = str(self.blas)
        self.chunks = split_chunks(data, n_chunks)[:self.P]
        self.wl, self.path = wl, path
        self.pool = mp.get_context("fork").Pool(self.P)

    def step(self, n_tokens):
        """one timed pass: every worker runs its chunk's first n_tokens; wall seconds."""
        jobs = [(str(self.path), ch, n_tokens, self.wl.window, self.wl.slide, self.wl.cdf_bits, self.blas)
                for ch in self.chunks]
        t0 = time.perf_counter()
        res = self.pool.map(_oracle_worker, jobs)
        dt = time.perf_counter() - t0
        return sum(r[0] for r in res), sum(r[1] for r in res), dt

    def sample(self, n_tokens):
        return (f"first {n_tokens} tokens of each of the first {self.P} chunks, one oracle process per chunk "
                f"({self.P} processes x {self.blas} BLAS threads): blocked fp64 {self.wl.shape} LM + walk + WNC")

    def close(self):
        self.pool.terminate()


def relaunch(args):
    """--gpus N > 1 outside torchrun: run this script under torch.distributed.run, N ranks."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def dry_run(args, wl, rank, world):
    """--dry-run (CPU, gloo): the launcher, rendezvous, shard plan, byte accounting and the
    max-over-ranks reduction of a GPU run, without a GPU or the model (tests/test_bench_contract)."""
    import torch
    import torch.distributed as dist
    import paper_2602_19626_b200 as nc
    from synth import make_text
    if world > 1:
        dist.init_process_group("gloo", init_method="env://")
    n_bytes = min(wl.n_bytes, 200_000)
    data = make_text(wl.text_kind, n_bytes * (1 if wl.name == "config3" else world), wl.text_seed)
    n_chunks = wl.n_chunks * world
    cuts = nc.nc_host_split(data, n_chunks)
    c0, c1 = nc.nc_host_shard_range(len(cuts) - 1, world, rank)
    mine = cuts[c1] - cuts[c0] if c1 > c0 else 0
    t = torch.tensor([float(mine), 1.0 + rank], dtype=torch.float64)
    tot = torch.tensor([float(mine)], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t[1:], op=dist.ReduceOp.MAX)
        dist.all_reduce(tot)
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "workload": wl.name, "scaling": scaling_of(wl),
                          "chunks": len(cuts) - 1, "bytes": len(data), "bytes_sum_over_ranks": int(tot.item()),
                          "max_over_ranks": float(t[1].item())}))
    if world > 1:
        dist.destroy_process_group()


def scaling_of(wl):
    return "strong" if wl.name == "config3" else "weak"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="config3")
    ap.add_argument("--no-decompress", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dry-run", action="store_true", help="CPU/gloo launcher + plan check (no GPU)")
    ap.add_argument("--oracle-tokens", type=int, default=192,
                    help="tokens per chunk per --impl reference step (chunk-parallel)")
    ap.add_argument("--baseline-tokens", type=int, default=1536, help="tokens per chunk of the cpu_baseline sample")
    ap.add_argument("--decompress-bytes", type=int, default=20000,
                    help="decompress sample: the first B bytes of every chunk of this rank (0 = the whole input)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    rank, world, local = dist_env()

    from synth import SHAPES, WORKLOADS, ensure_model, ensure_text, make_text
    wl = WORKLOADS[args.workload]
    metric, unit = "compress_bytes_per_sec", "B/s"
    if args.dry_run:
        return dry_run(args, wl, rank, world)

    if args.impl == "reference":
        if rank != 0:
            return
        path = ensure_model(wl.shape)
        data = open(ensure_text(args.workload), "rb").read()
        op = OraclePool(path, data, wl, wl.n_chunks)
        times, nb, ntk = [], 0, 0
        try:
            for i in range(args.warmup + args.steps):
                nb, ntk, dt = op.step(args.oracle_tokens)
                if i >= args.warmup:
                    times.append(dt)
        finally:
            op.close()
        v = nb * len(times) / sum(times)
        line = {"impl": "reference", "metric": metric, "value": v, "unit": unit, "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * statistics.mean(times),
                "higher_is_better": True, "scaling": scaling_of(wl), "vs_baseline": None, "dtype": "f64",
                "data": "synthetic", "config": {"workload": args.workload, "model": wl.shape,
                                                "sample": op.sample(args.oracle_tokens)},
                "cpu_baseline": {"value": v, "unit": unit, "cores": op.cores, "kind": "oracle",
                                 "sample": op.sample(args.oracle_tokens) + f" ({ntk} tokens, {nb} B per step)"},
                "e2e": {"value": v, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    import torch
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    if rank == 0:
        import __graft_entry__
        __graft_entry__.build()
        path = ensure_model(wl.shape)
        ensure_text(args.workload)
    if world > 1:
        dist.barrier()
    import paper_2602_19626_b200 as nc
    path = ensure_model(wl.shape)
    # config3: strong scaling (the same 10 MB at every N, wl.n_chunks chunks per rank);
    # otherwise weak scaling (each rank owns wl.n_bytes of input and wl.n_chunks chunks)
    strong = scaling_of(wl) == "strong"
    data = open(ensure_text(args.workload), "rb").read() if (world == 1 or strong) else \
        make_text(wl.text_kind, wl.n_bytes * world, wl.text_seed)
    n_chunks = wl.n_chunks * world
    prm = nc.nc_params_default(window=wl.window, slide=wl.slide, n_chunks=n_chunks, cdf_bits=wl.cdf_bits)
    model = nc.Model(path, local)
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream

    cuts = nc.nc_host_split(data, n_chunks)
    nch = len(cuts) - 1
    c0, c1 = nc.nc_host_shard_range(nch, world, rank)
    my_bytes = cuts[c1] - cuts[c0] if c1 > c0 else 0
    toks, ntok = [], []
    for c in range(c0, c1):
        t, _ = nc.nc_tokenize(model, data[cuts[c]:cuts[c + 1]], 1)
        toks.append(t)
        ntok.append(len(t))
    tokens = np.concatenate(toks) if toks else np.zeros(0, np.uint32)
    tok_dev = torch.from_numpy(tokens.view(np.int32).copy()).to(f"cuda:{local}")
    my_chunks = c1 - c0
    my_prm = nc.nc_params_default(window=wl.window, slide=wl.slide, n_chunks=max(1, c1 - c0), cdf_bits=wl.cdf_bits)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=f"cuda:{local}")   # > 126 MB L2

    def run_value():
        return nc.nc_compress_tokens(model, tok_dev.data_ptr(), np.array(ntok, np.uint32), my_prm, sptr)

    def timed(fn, k, w_, profile=False, clocks=None):
        for _ in range(w_):
            fn()
        total = 0.0
        launches = 0
        if profile:
            nc.nc_set_profiling(True)
        if clocks:
            clocks.start()
        out = None
        for _ in range(k):
            flush.zero_()
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            out = fn()
            e1.record(stream)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            total += e0.elapsed_time(e1)
            launches += nc.nc_last_stats()["kernel_launches"]
        clk = clocks.stop() if clocks else None
        prof = nc.nc_profile() if profile else None
        if profile:
            nc.nc_set_profiling(False)
        if world > 1:
            t = torch.tensor([total], dtype=torch.float64, device=f"cuda:{local}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            total = float(t.item())
        return total / 1000.0, out, launches // max(1, k), prof, clk

    # ---- value: device-resident tokens
    clocks = Clocks(local)
    t_val, blob_part, launches, _, clk = timed(run_value, args.steps, args.warmup, clocks=clocks)
    # per-kernel-class device time (roofline, breakdown): a separate pass with the library's
    # CUDA events around every launch, so the timed value above carries no profiling overhead
    n_prof = min(args.steps, 2)
    _, _, _, prof, _ = timed(run_value, n_prof, 0, profile=True)
    total_bytes = len(data)
    value = total_bytes * args.steps / t_val

    # ---- e2e: host bytes in, container (part) out, through the public API
    if world == 1:
        def run_e2e():
            return nc.nc_compress(model, data, prm, sptr)
    else:
        uid = nc.Comm.unique_id() if rank == 0 else bytes(128)
        obj = [uid]
        dist.broadcast_object_list(obj, src=0)
        comm = nc.Comm(rank, world, obj[0], local)

        def run_e2e():
            return nc.nc_compress_shard(model, comm, data, prm, sptr)
    t_e2e, e2e_out, _, _, _ = timed(run_e2e, args.steps, max(1, args.warmup // 2))
    e2e = total_bytes * args.steps / t_e2e

    # ---- correctness + bpb (N = 1: the e2e container round-trips) + decompress throughput.
    # Decoding is sequential per chunk (one token per chunk per step), so the whole 10 MB
    # would take minutes: the timed sample is the first --decompress-bytes of every chunk
    # (all 64 chunks decode in lockstep, ~4K tokens each = two window lengths, so the steps
    # reach the steady-state context), compressed and then decompressed through the public API.
    blob = e2e_out if world == 1 else None
    bpb, dec = None, None
    if world == 1:
        bpb = 8.0 * len(blob) / len(data)
        assert blob == blob_part, "device-resident and host-bytes paths disagree"
        if not args.no_decompress:
            if args.decompress_bytes:
                sub = b"".join(data[cuts[c]:min(cuts[c + 1], cuts[c] + args.decompress_bytes)] for c in range(nch))
                sprm = nc.nc_params_default(window=wl.window, slide=wl.slide, n_chunks=nch, cdf_bits=wl.cdf_bits)
                sblob = nc.nc_compress(model, sub, sprm, sptr)
            else:
                sub, sprm, sblob = data, prm, blob
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            back = nc.nc_decompress(model, sblob, sprm, sptr)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            assert back == sub, "round trip failed"
            dec = {"value": len(sub) / dt, "unit": "B/s", "seconds": dt, "bytes": len(sub), "chunks": nch,
                   "sample": (f"first {args.decompress_bytes} B of each of the {nch} chunks" if args.decompress_bytes
                              else "whole input"), "tokens_per_s": None}
            try:
                tk_sub, _ = nc.nc_tokenize(model, sub, nch)
                dec["tokens_per_s"] = len(tk_sub) / dt
            except Exception:
                pass
        else:
            assert len(blob) > 0

    # ---- roofline of the dominant kernel class (live CUDA events over the timed region)
    pk, pk_kind = peaks()
    kernels = {}
    for name, r in (prof or {}).items():
        if r["launches"]:
            kernels[name] = {"launches": r["launches"] // n_prof, "ms_per_step": r["ms"] / n_prof,
                             "work_per_step": r["work"] / n_prof}
    flop_classes = {"gemm_qkv", "gemm_o", "gemm_gateup", "gemm_down", "gemm_head", "attention"}
    # 3xTF32 on tcgen05: algorithmic FLOPs run as 3 tf32 MMAs; tf32 dense = bf16 dense / 2
    # (B200_PROFILING.md nominal ratio).  Kernels are timed inside a long step -> sustained peak.
    tc_peak = float(pk.get("bf16_tflops_sustained", pk["bf16_tflops"])) / 2.0 / 3.0
    # dominant kernel = largest share of the GPU's SM-time.  Every forward kernel runs on
    # all SMs; the walk holds one thread-block cluster per chunk (walk_ctas_per_chunk SMs)
    # and overlaps the next slab's forward, so its device time alone overstates its share.
    walk_sms = min(N_SM, my_chunks * nc.nc_host_walk_ctas(SHAPES[wl.shape].vocab, my_chunks)) if my_chunks else N_SM
    sm_share = {k: kernels[k]["ms_per_step"] * (walk_sms if k == "walk" else N_SM) for k in kernels}
    dom = max(kernels, key=lambda k: sm_share[k]) if kernels else None
    roof = None
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            traffic = json.load(f).get(dom)
    except Exception:
        pass
    if dom:
        r = kernels[dom]
        per_launch_ms = r["ms_per_step"] / max(1, r["launches"])
        work_launch = r["work_per_step"] / max(1, r["launches"])
        if dom in flop_classes:
            ach = work_launch / (per_launch_ms / 1e3) / 1e12
            roof = {"kernel": dom, "bound": "tensor", "achieved": ach, "peak": tc_peak, "unit": "TFLOP/s",
                    "frac": ach / tc_peak, "traffic": traffic,
                    "peak_source": f"{pk_kind} bf16 sustained {pk.get('bf16_tflops_sustained')} TF/s / 2 (tf32) / 3 "
                                   "(3xTF32 passes), algorithmic FLOPs"}
        else:
            ach = work_launch / (per_launch_ms / 1e3) / 1e9
            roof = {"kernel": dom, "bound": "hbm", "achieved": ach, "peak": pk["hbm_gbs"], "unit": "GB/s",
                    "frac": ach / pk["hbm_gbs"], "traffic": traffic, "peak_source": pk_kind}
        roof["share_of_step"] = r["ms_per_step"] / (1000 * t_val / args.steps)
    walk = kernels.get("walk")
    if walk:
        kernels["walk"]["hbm_gbs"] = walk["work_per_step"] / (walk["ms_per_step"] / 1e3) / 1e9
        kernels["walk"]["hbm_frac"] = kernels["walk"]["hbm_gbs"] / pk["hbm_gbs"]
        kernels["walk"]["sms"] = walk_sms
        kernels["walk"]["us_per_token_per_chunk"] = 1e3 * walk["ms_per_step"] / max(1, max(ntok) if ntok else 1)
    for k in kernels:
        kernels[k]["sm_time_share"] = sm_share[k] / (N_SM * 1000 * t_val / args.steps)
    for k in flop_classes & set(kernels):
        kernels[k]["tflops"] = kernels[k]["work_per_step"] / (kernels[k]["ms_per_step"] / 1e3) / 1e12

    # ---- fused roofline of the whole step: the algorithmic FLOPs of the
    # forward at the 3xTF32 sustained tensor rate plus the walk's 8V bytes per token (logits
    # written by the head, read by the walk) at measured HBM bandwidth, against the step time
    fused = None
    if kernels and flop_classes & set(kernels):
        f_step = sum(kernels[k]["work_per_step"] for k in flop_classes & set(kernels))
        b_step = 8.0 * SHAPES[wl.shape].vocab * float(sum(ntok))
        t_roof = f_step / (tc_peak * 1e12) + b_step / (pk["hbm_gbs"] * 1e9)
        fused = {"flop_per_step": f_step, "bytes_per_step": b_step, "ms_roofline": 1e3 * t_roof,
                 "frac": t_roof / (t_val / args.steps),
                 "peaks": f"{tc_peak:.1f} TFLOP/s (3xTF32 sustained), {pk['hbm_gbs']:.0f} GB/s"}

    # ---- CPU oracle baseline (rank 0, N = 1 only, bounded sample)
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        op = OraclePool(path, data, wl, n_chunks)
        try:
            nb, ntk, dt = op.step(args.baseline_tokens)
        finally:
            op.close()
        cpu = {"value": nb / dt, "unit": unit, "cores": op.cores, "kind": "oracle",
               "sample": op.sample(args.baseline_tokens) + f": {ntk} tokens, {nb} B in {dt:.1f} s"}

    n_tok_total = int(sum(ntok))
    if world > 1:
        t = torch.tensor([n_tok_total], dtype=torch.int64, device=f"cuda:{local}")
        dist.all_reduce(t)
        n_tok_total = int(t.item())
    if rank == 0:
        line = {
            "metric": metric, "value": value, "unit": unit, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000 * t_val / args.steps, "higher_is_better": True,
            "scaling": scaling_of(wl), "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": args.workload, "model": wl.shape, "text": wl.text_kind,
                       "bytes_total": len(data), "chunks_total": nch,
                       "bytes_per_gpu": my_bytes, "chunks_per_gpu": my_chunks, "window": wl.window,
                       "slide": wl.slide, "cdf_bits": wl.cdf_bits, "tokens": n_tok_total,
                       "l2": "256 MB buffer written between timed steps; working set (538 MB weights, "
                             "logit slabs) > 126 MB L2",
                       "parallelism": f"chunk-sharded x{world}"},
            "e2e": {"value": e2e, "unit": unit, "h2d_bytes_per_step": 4 * n_tok_total,
                    "d2h_bytes_per_step": 8 * n_tok_total},
            "gpu_launches": launches,
            "roofline": roof,
            "fused_roofline": fused,
            "cpu_baseline": cpu,
            "clocks": clk,
            "bpb": bpb,
            "decompress": dec,
            "kernels": kernels,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
