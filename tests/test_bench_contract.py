"""CPU test of bench.py's reference arm (the CPU oracle as the reference, ③/④): it runs
without a GPU and prints one JSON line with the contract's keys."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0", "--oracle-tokens", "16"], capture_output=True, text=True, timeout=600,
                       cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["metric"] == "compress_bytes_per_sec" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["value"] == line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert line["config"]["workload"] == "config3" and line["scaling"] == "strong"
    assert line["cpu_baseline"]["cores"] >= 1 and "chunks" in line["cpu_baseline"]["sample"]


def test_launcher_dry_run_world2():
    """`bench.py --gpus 2` outside torchrun re-launches itself under torch.distributed.run with
    two ranks (here on CPU with gloo, --dry-run): rendezvous on 127.0.0.1, the shard plan of
    the default workload (config3: strong scaling, 64 chunks per rank), the byte accounting
    over ranks and the max-over-ranks reduction; rank 0 alone prints one JSON line."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["dry_run"] and d["n_gpus"] == 2 and d["workload"] == "config3" and d["scaling"] == "strong"
    assert d["chunks"] == 128 and d["bytes_sum_over_ranks"] == d["bytes"]
    assert d["max_over_ranks"] == 2.0
