"""bench.py --gpus N launches N ranks by itself (`--gpus` was parsed
and never used). On CPU the launcher self-test runs the same re-exec under
torch.distributed.run with gloo: every rank joins and rank 0 prints one line."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(n):
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR",
                                                             "MASTER_PORT")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--launch-check"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_bench_gpus_2_launches_two_ranks():
    out = _run(2)
    assert out["n_gpus"] == 2 and out["ranks"] == [0, 1] and out["backend"] == "gloo"


def test_bench_gpus_1_stays_single_process():
    out = _run(1)
    assert out["n_gpus"] == 1 and out["ranks"] == [0]
