"""Summarise ncu outputs from gpurun_out/ into profiles/ (tracked).

  python tools/ncu_summary.py <round tag, e.g. r01> [launches.csv] [name=report.ncu-rep ...]

Writes profiles/<tag>_launches.md (per-kernel share of the step from the
gpu__time_duration launch list), profiles/<tag>_<name>.md (key --set full
metrics per captured launch) and profiles/ncu_traffic.json (DRAM bytes per
launch by kernel class, read by bench.py for roofline.traffic)."""
import collections
import csv
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "l1tex__t_bytes.sum", "lts__t_bytes.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__cluster_dim_x", "sm__cycles_elapsed.avg.per_second"]
CLASS = {"attention_kernel": "attention", "walk_kernel": "walk", "attn_tc_kernel": "attention",
         "walk_cl_kernel<4>": "walk", "nc::walk_cl_kernel<(int)4>": "walk", "walk_cl_kernel<8>": "walk",
         "nc::walk_cl_kernel<(int)8>": "walk", "nc::attn_tc_kernel": "attention", "gemm_tc_kernel<0>": "gemm_qkv",
         "gemm_tc_kernel<1>": "gemm_o|gemm_down", "gemm_tc_kernel<2>": "gemm_gateup", "gemm_tc_kernel<3>": "gemm_head",
         "nc::gemm_tc_kernel<0>": "gemm_qkv", "nc::gemm_tc_kernel<1>": "gemm_o|gemm_down",
         "nc::gemm_tc_kernel<2>": "gemm_gateup", "nc::gemm_tc_kernel<3>": "gemm_head",
         "ngram_pre_kernel": "ngram", "nc::ngram_pre_kernel": "ngram"}


def to_ns(v, u):
    v = float(v.replace(",", ""))
    return v * {"ns": 1, "nsecond": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}.get(u, 1)


def launches(tag, path):
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if r and r[0] == "ID")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if len(r) != len(hdr) or r[0] == "ID":
            continue
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"].split("(")[0].replace("void ", "")
        agg[k][0] += 1
        agg[k][1] += to_ns(d["Metric Value"], d["Metric Unit"])
    tot = sum(v[1] for v in agg.values())
    lines = [f"# {tag}: ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)",
             f"source: {os.path.basename(path)}; {sum(v[0] for v in agg.values())} launches", "",
             "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| {k} | {n} | {t / 1e6:.2f} | {t / tot:.1%} |")
    open(os.path.join(PROF, f"{tag}_launches.md"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def full(tag, name, rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    lines = [f"# {tag}: ncu --set full, {name} ({os.path.basename(rep)})", ""]
    traffic = {}
    seen = {}
    for r in rows[2:]:
        kn = r[idx["Kernel Name"]]
        lines.append(f"## {kn}")
        for k in KEYS:
            if k in idx:
                lines.append(f"- {k} = {r[idx[k]]} {units[idx[k]]}")
        rd = float(r[idx["dram__bytes_read.sum"]].replace(",", "")) * (1e6 if units[idx["dram__bytes_read.sum"]] == "Mbyte" else 1e3 if units[idx["dram__bytes_read.sum"]] == "Kbyte" else 1e9 if units[idx["dram__bytes_read.sum"]] == "Gbyte" else 1)
        wr = float(r[idx["dram__bytes_write.sum"]].replace(",", "")) * (1e6 if units[idx["dram__bytes_write.sum"]] == "Mbyte" else 1e3 if units[idx["dram__bytes_write.sum"]] == "Kbyte" else 1e9 if units[idx["dram__bytes_write.sum"]] == "Gbyte" else 1)
        base = kn.split("(")[0].replace("void ", "").strip()
        base = re.sub(r"gemm_tc_kernel<\(?\w*\)?(\d+), \(?\w*\)?\d+(, \(?\w*\)?\w+)?>", r"gemm_tc_kernel<\1>", base)
        if base.startswith("walk_cl_kernel") or base.startswith("nc::walk_cl_kernel"):
            base = "walk_cl_kernel<8>"
        alts = CLASS.get(base, base).split("|")   # several classes share a kernel: capture order
        k_ = seen.get(base, 0)
        seen[base] = k_ + 1
        traffic[alts[min(k_, len(alts) - 1)]] = rd + wr
        lines.append("")
    open(os.path.join(PROF, f"{tag}_{name}.md"), "w").write("\n".join(lines) + "\n")
    tpath = os.path.join(PROF, "ncu_traffic.json")
    cur = json.load(open(tpath)) if os.path.exists(tpath) else {}
    cur.update({k: v for k, v in traffic.items()})
    cur["_note"] = f"dram read+write bytes per launch from ncu --set full captures ({tag})"
    json.dump(cur, open(tpath, "w"), indent=1)


if __name__ == "__main__":
    os.makedirs(PROF, exist_ok=True)
    tag = sys.argv[1]
    for a in sys.argv[2:]:
        if "=" in a:
            n, p = a.split("=", 1)
            full(tag, n, p)
        else:
            launches(tag, a)
