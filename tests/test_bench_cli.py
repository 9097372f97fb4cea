"""bench.py's multi-rank launch without a GPU: `--gpus 2 --dry-run` re-executes itself under
torchrun (two ranks, gloo on 127.0.0.1), shards the C3 inventory and all-gathers per-rank
payloads shaped like the top-K keys; rank 0 prints one JSON line."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_gpus2_dry_run():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    rec = json.loads(lines[0])
    assert rec["dry_run"] and rec["n_gpus"] == 2 and rec["gather_ok"]
    assert rec["config"]["workload"].startswith("C3:")
    (a0, a1), (b0, b1) = rec["shards"]
    assert a0 == 0 and a1 == b0 and b1 == rec["config"]["n_ads"] and a1 % 128 == 0
