"""Trace ingestion on the GPU (csrc/sfk_trace.cu via workloads.load_trace)
against what the reference's load_trace made of the same files
(tests/golden/make_golden_traces.py): ops, keys, or the TraceFormatError's
line number and message. Newline conventions, str.strip whitespace, int(,10)
syntax, Unicode lines (finished on the host), and a 20k-op round trip."""

import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_1701_04148_b200 as P  # noqa: E402
from paper_1701_04148_b200 import workloads as W  # noqa: E402

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "traces")
EXPECTED = json.load(open(os.path.join(HERE, "expected.json")))


@pytest.mark.parametrize("name", sorted(EXPECTED))
def test_trace_matches_reference(name):
    want = EXPECTED[name]
    path = os.path.join(HERE, name + ".trace")
    if "error_line" in want:
        with pytest.raises(P.TraceFormatError) as exc:
            W.load_trace(path)
        assert exc.value.line_number == want["error_line"]
        assert str(exc.value) == want["message"]
    else:
        ops, keys = W.load_trace(path)
        np.testing.assert_array_equal(ops.cpu().numpy(), np.array(want["ops"], dtype=np.uint8))
        np.testing.assert_array_equal(keys.cpu().numpy(), np.array([int(k) for k in want["keys"]], dtype=np.uint64))


def test_read_trace_yields_prefix_then_raises():
    path = os.path.join(HERE, "bad_after_comments.trace")
    got = []
    with pytest.raises(P.TraceFormatError) as exc:
        for op in W.read_trace(path):
            got.append(op)
    assert got == [W.Operation("insert", 1)]
    assert exc.value.line_number == 4


def test_write_then_load_round_trip(tmp_path):
    rng = np.random.default_rng(3)
    keys = rng.integers(0, np.iinfo(np.uint64).max, size=50_000, dtype=np.uint64)
    ops = (rng.random(keys.size) < 0.25).astype(np.uint8)
    p = tmp_path / "rt.trace"
    W.write_trace(p, (W.Operation("delete" if o else "insert", int(k)) for o, k in zip(ops, keys)))
    o2, k2 = W.load_trace(p)
    np.testing.assert_array_equal(o2.cpu().numpy(), ops)
    np.testing.assert_array_equal(k2.cpu().numpy(), keys)


def test_trace_feeds_a_sketch(oracle):
    """The parsed device arrays go straight into apply_ops."""
    ops, keys = W.load_trace(os.path.join(HERE, "roundtrip.trace"))
    sk = P.SfSketch(P.SketchParams(d=4, w=512, z=4, master_seed=9), "sff")
    sk.apply_ops(ops, keys)
    o = oracle.OracleSketch("sff", 4, 512, 4, None, 9)
    st = o.apply_ops(ops.cpu().numpy(), keys.cpu().numpy())
    assert st[0] == 0
    np.testing.assert_array_equal(sk.slim.counters.cpu().numpy(), o.slim)
