"""`bench.py --gpus N` launches N ranks (one process per GPU on the box): the
relaunch under torch.distributed.run, the contiguous request shards and the
post-timing all_gather, rehearsed on CPU with gloo (--dry-run), world size 2."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_gpus2_dry_run_launches_two_ranks():
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--dry-run", "--batch", "8"], capture_output=True, text=True,
                         timeout=300, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1                       # rank 0 alone prints
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2
    assert rec["requests"] == 16 and rec["gathered_shape"] == [16, 6]
    assert rec["gathered_ok"] and rec["max_over_ranks"] == 2.0
