"""bench.py's launch contract on a host without GPUs (CPU): `--gpus N` never runs fewer ranks
than it reports — it re-launches itself one process per GPU, refuses when N GPUs are not
visible, and refuses a WORLD_SIZE that differs from N."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(args, env_extra=None):
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="", **(env_extra or {}))
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, env=env,
                          capture_output=True, text=True, timeout=300)


def test_gpus_more_than_visible_refused():
    r = run_bench(["--gpus", "2", "--steps", "1", "--warmup", "3"])
    assert r.returncode != 0
    assert "needs 2 visible GPUs, found 0" in r.stderr + r.stdout


def test_world_size_mismatch_refused():
    r = run_bench(["--gpus", "1", "--steps", "1", "--warmup", "3"],
                  {"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode != 0
    assert "--gpus 1 but WORLD_SIZE=2" in r.stderr + r.stdout
