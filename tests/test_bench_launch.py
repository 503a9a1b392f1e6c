"""bench.py's multi-rank launch on CPU: `python bench.py --gpus 2 --dry-run` without a torchrun
environment re-executes itself through torch.distributed.run (2 ranks, gloo); exactly one JSON line
(rank 0) comes back, with the max-over-ranks reduction and the particle shard of rank 0."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_self_launches_two_ranks():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR",
                                                              "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"], cwd=ROOT,
                       env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    j = json.loads(lines[0])
    assert j["dry_run"] and j["n_gpus"] == 2 and j["ranks_max"] == 2.0
    assert j["workload"] == "S1" and j["rows_rank0"] == [0, 32]
