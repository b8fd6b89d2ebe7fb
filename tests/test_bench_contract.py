"""bench.py's multi-rank contract on CPU: the reference arm runs on rank 0
only (other ranks exit 0 without work), N>1 defaults to north_star's layout
(build on rank 0, slim broadcast, sharded queries; strong scaling) with
independent replicas behind --replicas, and the reference arm times the
reference package from baseline/_ref when it is installed."""

import argparse
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def _args(**kw):
    a = argparse.Namespace(replicas=False, shared_slim=False, alpha=1.0, alpha_q=1.0, queries=1_000_000_000,
                           cpu_kind="auto")
    for k, v in kw.items():
        setattr(a, k, v)
    return a


def test_reference_arm_other_ranks_exit_without_work():
    env = dict(os.environ, WORLD_SIZE="2", RANK="1", LOCAL_RANK="1")
    p = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--gpus", "2", "--steps", "1",
                        "--warmup", "0"], cwd=ROOT, env=env, capture_output=True, text=True, timeout=120)
    assert p.returncode == 0, p.stderr
    assert p.stdout.strip() == ""


def test_broadcast_and_sharded_queries_is_the_multi_gpu_default():
    assert not bench.replicas(_args(), 1)
    assert not bench.replicas(_args(), 2)
    assert bench.replicas(_args(replicas=True), 8)
    cfg = bench.workload_config(_args(), 8)
    assert cfg["parallelism"].startswith("north_star layout: build on rank 0")
    assert "queries sharded contiguously over 8 GPUs" in cfg["parallelism"]
    assert bench.workload_config(_args(), 1)["parallelism"] == "1 GPU"
    rep = bench.workload_config(_args(replicas=True), 4)["parallelism"]
    assert rep.startswith("replicas only: 4 independent sketches") and "no data-path collective" in rep


def test_cpu_baseline_kind_prefers_the_installed_reference():
    kind, ref = bench.cpu_kind(_args())
    if os.path.isfile(os.path.join(ROOT, "baseline", "_ref", "sfsketch", "__init__.py")):
        assert kind == "reference" and ref is not None and hasattr(ref, "SfSketch")
    else:
        assert kind == "port" and ref is None
    assert bench.cpu_kind(_args(cpu_kind="port")) == ("port", None)


def test_reference_cpu_measure_matches_the_port_on_a_small_stream():
    """Both CPU arms (the reference package and the C port) build the same
    state and answer the same estimates on a small cfg-3-shaped stream."""
    from paper_1701_04148_b200 import workloads as Wl

    kind, ref = bench.cpu_kind(_args())
    if kind != "reference":
        import pytest

        pytest.skip("baseline/_ref not installed")
    st = Wl.cfg3(seed=3, n_ins=100_000, v=10_000, alpha=1.0)
    qs = Wl.query_keys(7, st["distinct"], 1.0, 0, 20_000)
    a = _args(queries=20_000)
    r = bench.cpu_measure(a, st, qs, 2, "reference", ref)
    p = bench.cpu_measure(a, st, qs, 2, "port", None)
    for x, y in zip(bench.cpu_state("reference", r[4]), bench.cpu_state("port", p[4])):
        assert (x == y).all()
    assert (r[5] == p[5]).all()
