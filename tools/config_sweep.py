"""Measure the BASELINE.json configs other than the bench workload on one
B200 and print one JSON object per line (diagnostics; needs a GPU).

  python tools/config_sweep.py [c5] [c2chunks]

c5       : config 5 on the config-2 input: compress B/s and bpb at L = 512 / 1024 / 2048
           (C = L/4, 8 chunks), CDF-16 vs CDF-24 (delta bits/token vs log2(T/(T-V))),
           and sequential decode (decompress) with 64 chunks at each window.
c2chunks : config 2 with 1 vs 8 chunks (compress B/s, bpb, walk us/token/chunk).
c3 [rows]: config 3 (10 MB, 64 chunks) with max_slab_rows = rows (default 32768); run under
           NC_WALK_CS=4|8 to compare walk cluster sizes (read once per process).
slabs    : config 2 (8 chunks) under explicit slab plans (NC_SLAB_PLAN), median of 5 with a
           256 MB L2 flush between runs: the first slab's 256-row tile count against the
           74 CTA pairs of the GEMMs vs the length of the last slab's walk.
Configs 3 and 4 run through bench.py (--workload config3 / config4_shard).
Timing: CUDA events on the launching stream around nc_compress_tokens (device-resident
token ids, like bench.py's value), median of 3 after 1 warm-up; decompress: wall clock of
nc_decompress (host bytes in and out), one run after one warm-up of compress.
"""
import json
import math
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import __graft_entry__  # noqa: E402

__graft_entry__.build()
import paper_2602_19626_b200 as nc  # noqa: E402
from synth import WORKLOADS, ensure_model, ensure_text  # noqa: E402

model = nc.Model(ensure_model("smollm2-135m"), 0)
stream = torch.cuda.current_stream()
V = 49152


def tokens_dev(data, n_chunks):
    cuts = nc.nc_host_split(data, n_chunks)
    toks, ntok = [], []
    for c in range(len(cuts) - 1):
        t, _ = nc.nc_tokenize(model, data[cuts[c]:cuts[c + 1]], 1)
        toks.append(t)
        ntok.append(len(t))
    tok = np.concatenate(toks)
    return torch.from_numpy(tok.view(np.int32).copy()).cuda(), ntok


_flush = None


def compress_timed(data, prm, n_chunks, reps=3, flush=False):
    global _flush
    if flush and _flush is None:
        _flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    td, ntok = tokens_dev(data, n_chunks)
    f = lambda: nc.nc_compress_tokens(model, td.data_ptr(), np.array(ntok, np.uint32), prm, stream.cuda_stream)
    f()
    ts = []
    blob = None
    for _ in range(reps):
        if flush:
            _flush.fill_(1)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        blob = f()
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
        st = nc.nc_last_stats()
    return statistics.median(ts), blob, int(sum(ntok)), st


def line(**kw):
    print(json.dumps(kw), flush=True)


args = set(a for a in sys.argv[1:] if not a.isdigit()) or {"c5", "c2chunks"}
nums = [int(a) for a in sys.argv[1:] if a.isdigit()]
data2 = open(ensure_text("config2"), "rb").read()

if "c2chunks" in args:
    for n_chunks in (1, 8):
        prm = nc.nc_params_default(window=2048, slide=512, n_chunks=n_chunks)
        t, blob, ntok, st = compress_timed(data2, prm, n_chunks)
        line(config="config2", chunks=n_chunks, bytes=len(data2), tokens=ntok, compress_Bps=len(data2) / t,
             ms=1e3 * t, bpb=8.0 * len(blob) / len(data2),
             walk_us_per_token_per_chunk=1e3 * st["walk_ms"] / (ntok / n_chunks))

if "c3" in args:
    data3 = open(ensure_text("config3"), "rb").read()
    rows = nums[0] if nums else 32768
    prm = nc.nc_params_default(window=2048, slide=512, n_chunks=64, max_slab_rows=rows)
    t, blob, ntok, st = compress_timed(data3, prm, 64, reps=2, flush=True)
    line(config="config3", chunks=64, max_slab_rows=rows, walk_cs=os.environ.get("NC_WALK_CS", "default"),
         compress_Bps=len(data3) / t, ms=1e3 * t, bytes=len(blob))

if "slabs" in args:
    prm = nc.nc_params_default(window=2048, slide=512, n_chunks=8)
    for plan in ("", "2944", "3072", "3200", "3328", "3456", "3584", "3072,640", "2560,1024"):
        if plan:
            os.environ["NC_SLAB_PLAN"] = plan
        else:
            os.environ.pop("NC_SLAB_PLAN", None)
        t, blob, ntok, st = compress_timed(data2, prm, 8, reps=5, flush=True)
        line(config="config2", chunks=8, slab_plan=plan or "default", compress_Bps=len(data2) / t, ms=1e3 * t,
             bytes=len(blob))
    os.environ.pop("NC_SLAB_PLAN", None)

if "c5" in args:
    bits = {}
    for wl_name in ("config5_l512", "config5_l1024", "config2", "config5_cdf16"):
        wl = WORKLOADS[wl_name]
        prm = nc.nc_params_default(window=wl.window, slide=wl.slide, n_chunks=wl.n_chunks, cdf_bits=wl.cdf_bits)
        t, blob, ntok, st = compress_timed(data2, prm, wl.n_chunks)
        bits[wl_name] = (len(blob), ntok)
        line(config="config5", workload=wl_name, window=wl.window, slide=wl.slide, cdf_bits=wl.cdf_bits,
             chunks=wl.n_chunks, tokens=ntok, compress_Bps=len(data2) / t, ms=1e3 * t,
             bpb=8.0 * len(blob) / len(data2))
    n24, tk = bits["config2"]
    n16, _ = bits["config5_cdf16"]
    hdr = 9 + 12 * WORKLOADS["config2"].n_chunks
    line(config="config5", cdf16_vs_cdf24_delta_bits_per_token=8.0 * (n16 - n24) / tk,
         predicted_upper=math.log2(2 ** 16 / (2 ** 16 - V)), predicted_cdf24=math.log2(2 ** 24 / (2 ** 24 - V)),
         container_bytes={"cdf24": n24, "cdf16": n16, "header_and_table": hdr})
    for L in (512, 1024, 2048):
        prm = nc.nc_params_default(window=L, slide=L // 4, n_chunks=64)
        blob = nc.nc_compress(model, data2, prm, stream.cuda_stream)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        back = nc.nc_decompress(model, blob, prm, stream.cuda_stream)
        dt = time.perf_counter() - t0
        assert back == data2, "round trip failed"
        _, ntok = tokens_dev(data2, 64)
        line(config="config5", decode_window=L, chunks=64, tokens=int(sum(ntok)), steps=max(ntok),
             decompress_Bps=len(data2) / dt, decode_tokens_per_s=sum(ntok) / dt, seconds=dt,
             ms_per_step=1e3 * dt / max(ntok))
