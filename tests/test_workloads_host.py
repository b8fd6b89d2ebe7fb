"""Host-side pieces of the workload API, CPU only: WorkloadSpec validation
(the reference's rules and messages, workloads.py:58-73), the per-line trace
rules the host applies to non-ASCII lines and error messages
(workloads.py:137-155) replayed over the reference-generated trace fixtures,
and write_trace's format."""

import json
import os

import numpy as np
import pytest

from paper_1701_04148_b200 import errors as E
from paper_1701_04148_b200 import workloads as W

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "traces")


@pytest.mark.parametrize("kwargs,msg", [
    (dict(kind="poisson"), "unknown workload kind 'poisson'"),
    (dict(kind="trace"), "trace workloads need trace_path"),
    (dict(kind="zipf", distinct_items=0, total_ops=5), "distinct_items must be >= 1"),
    (dict(kind="zipf", distinct_items=5, total_ops=-1), "total_ops must be >= 0"),
    (dict(kind="zipf", distinct_items=5, total_ops=5, zipf_skew=0.0), "zipf_skew must be > 0"),
    (dict(kind="uniform", distinct_items=5, total_ops=5, deletion_mode="random"), "unknown deletion mode 'random'"),
    (dict(kind="uniform", distinct_items=5, total_ops=5, deletion_mode="interleaved", delete_prob=1.0),
     "interleaved delete_prob must lie in [0, 1)"),
])
def test_spec_validation(kwargs, msg):
    with pytest.raises(E.ConfigurationError) as exc:
        W.WorkloadSpec(**kwargs)
    assert str(exc.value) == msg


def test_spec_is_immutable():
    s = W.WorkloadSpec(kind="zipf", distinct_items=3, total_ops=4)
    with pytest.raises(AttributeError):
        s.total_ops = 5


def _host_parse(path):
    """The host line rules over a whole file (Python's universal newlines)."""
    ops, keys = [], []
    with open(path, "r", encoding="utf-8") as fh:
        for lineno, line in enumerate(fh, start=1):
            r = W._trace_line(line, lineno)
            if r is not None:
                ops.append(r[0])
                keys.append(r[1])
    return ops, keys


@pytest.mark.parametrize("name", sorted(json.load(open(os.path.join(HERE, "expected.json")))))
def test_host_line_rules_match_reference(name):
    want = json.load(open(os.path.join(HERE, "expected.json")))[name]
    path = os.path.join(HERE, name + ".trace")
    if "error_line" in want:
        with pytest.raises(E.TraceFormatError) as exc:
            _host_parse(path)
        assert str(exc.value) == want["message"]
        assert exc.value.line_number == want["error_line"]
    else:
        ops, keys = _host_parse(path)
        assert ops == want["ops"]
        assert [str(k) for k in keys] == want["keys"]


def test_write_trace_format(tmp_path):
    p = tmp_path / "w.trace"
    W.write_trace(p, [W.Operation("insert", 5), W.Operation("delete", 2**64 - 1)])
    assert p.read_bytes() == b"I,5\nD,18446744073709551615\n"


def test_zipf_probabilities_sum_to_one():
    p = W.zipf_probabilities(1000, 1.2)
    assert p.shape == (1000,) and abs(p.sum() - 1.0) < 1e-12 and np.all(np.diff(p) < 0)
