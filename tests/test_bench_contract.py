"""bench.py's multi-rank contract on CPU: the reference arm runs on rank 0
only (other ranks exit 0 without work), and N>1 defaults to one independent
replica per GPU (weak scaling, no data-path collective)."""

import argparse
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def _args(**kw):
    a = argparse.Namespace(shared_slim=False, alpha=1.0, alpha_q=1.0, queries=1_000_000_000)
    for k, v in kw.items():
        setattr(a, k, v)
    return a


def test_reference_arm_other_ranks_exit_without_work():
    env = dict(os.environ, WORLD_SIZE="2", RANK="1", LOCAL_RANK="1")
    p = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--gpus", "2", "--steps", "1",
                        "--warmup", "0"], cwd=ROOT, env=env, capture_output=True, text=True, timeout=120)
    assert p.returncode == 0, p.stderr
    assert p.stdout.strip() == ""


def test_replicas_is_the_multi_gpu_default():
    assert not bench.replicas(_args(), 1)
    assert bench.replicas(_args(), 2)
    assert not bench.replicas(_args(shared_slim=True), 8)
    cfg = bench.workload_config(_args(), 8)
    assert cfg["parallelism"].startswith("replicas only: 8 independent sketches")
    assert "no data-path collective" in cfg["parallelism"]
    assert bench.workload_config(_args(), 1)["parallelism"] == "1 GPU"
    assert "queries sharded over 4" in bench.workload_config(_args(shared_slim=True), 4)["parallelism"]
