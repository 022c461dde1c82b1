"""bench.py's multi-rank plumbing on CPU (`--gpus N` must start N ranks by itself).

`python bench.py --gpus 2 --dry-run` has no torchrun environment, so bench.py re-launches itself under
torch.distributed.run with 2 ranks (gloo here); rank 0 alone prints ONE JSON line with n_gpus = 2,
the step time being the max over ranks, and N > 1 defaults to the row-sharded C5 model."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_spawns_ranks_and_prints_one_line():
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR",
                                                             "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run", "--steps", "3",
                        "--warmup", "3"], capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 3
    assert d["config"]["model"] == "llama3-70b" and d["config"]["parallelism"] == "tp2"
