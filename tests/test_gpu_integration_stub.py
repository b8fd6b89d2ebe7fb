"""The reference-side ctypes binding printed in INTEGRATION.md (the stub a
maintainer would add as sfsketch/_kernels_b200.py) is executed as written —
only its library path is pointed at the in-tree build — and its
sf_bucket_apply / min_query / count_apply are checked against the oracle's
restatement of _kernels.sf_bucket_apply, min_query and count_apply
(_kernels.py:318-384, 229-241, 118-146) with the reference's own argument
conventions: device counters mutated in place, the reference's status tuple
returned, estimates written into a host numpy `out`."""

import os
import re

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_1701_04148_b200 import _lib  # noqa: E402
from paper_1701_04148_b200.hashing import seed_array  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def stub_with(name):
    """Exec the INTEGRATION.md block defining `name` (after the block that
    opens the library, when that is another block) in one namespace."""
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    blocks = [blk.replace("/path/to/paper_1701_04148_b200/_lib/libsfsketch_cuda.so", _lib.LIB_PATH)
              for blk in re.findall(r"```python\n(.*?)```", text, re.S)]
    opener = next(blk for blk in blocks if "_L = ctypes.CDLL(" in blk)
    target = next((blk for blk in blocks if f"def {name}(" in blk), None)
    assert target is not None, f"INTEGRATION.md has no binding for {name}"
    ns = {}
    if target is not opener:
        exec(compile(opener, "INTEGRATION.md", "exec"), ns)
    exec(compile(target, "INTEGRATION.md", "exec"), ns)
    return ns


@pytest.mark.parametrize("mode", [0, 1])
def test_stub_sf_bucket_apply_and_min_query(oracle, mode):
    ns = stub_with("sf_bucket_apply")
    rng = np.random.default_rng(mode)
    d, w, z, n = 4, 4096, 4, 200_000
    bseeds, sseeds = seed_array(21, 0, d), seed_array(21, d, d)
    vocab = rng.integers(0, 1 << 63, size=5000, dtype=np.uint64)
    keys = vocab[np.minimum(rng.zipf(1.2, size=n) - 1, vocab.size - 1)]
    ops = np.zeros(n, np.uint8)
    ops[n // 2:][rng.random(n - n // 2) < 0.15] = 1
    # deletes only of keys inserted earlier (a valid stream)
    dels = np.nonzero(ops)[0]
    ops[dels] = 0
    ins_idx = np.nonzero(ops == 0)[0]
    ops[dels] = 1
    keys[dels] = keys[rng.choice(ins_idx[ins_idx < n // 2], size=dels.size)]
    slim = torch.zeros((d, w), dtype=torch.uint32, device="cuda")
    fat = torch.zeros((d, w, z), dtype=torch.uint32, device="cuda")
    inc = torch.zeros(d, dtype=torch.int64, device="cuda")
    st = ns["sf_bucket_apply"](slim, fat, bseeds, sseeds, mode, ops, keys, inc)
    o_slim = np.zeros((d, w), np.uint32)
    o_fat = np.zeros((d, w, z), np.uint32)
    o_inc = np.zeros(d, np.int64)
    o_st = oracle.sf_bucket_apply(o_slim, o_fat, bseeds, sseeds, mode, ops, keys, o_inc)
    assert tuple(st) == tuple(o_st)
    np.testing.assert_array_equal(slim.cpu().numpy(), o_slim)
    np.testing.assert_array_equal(fat.cpu().numpy(), o_fat)
    np.testing.assert_array_equal(inc.cpu().numpy(), o_inc)
    q = np.concatenate([vocab, rng.integers(0, 1 << 63, size=20_000, dtype=np.uint64)])
    out = np.empty(q.size, np.int64)
    ns["min_query"](slim, bseeds, q, out)
    np.testing.assert_array_equal(out, oracle.min_query(o_slim, bseeds, q))


def test_stub_count_apply(oracle):
    ns = stub_with("count_apply")
    rng = np.random.default_rng(5)
    d, w, n = 3, 2048, 50_000
    seeds = seed_array(8, 0, d)  # Count: one seed per row (the sign uses a salted hash of it)
    keys = rng.integers(0, 3000, size=n).astype(np.uint64)
    ops = np.zeros(n, np.uint8)
    counters = torch.zeros((d, w), dtype=torch.int32, device="cuda")
    st = ns["count_apply"](counters, seeds, ops, keys)
    o = np.zeros((d, w), np.int32)
    o_st = oracle.count_apply(o, seeds, ops, keys)
    assert tuple(st) == tuple(o_st)
    np.testing.assert_array_equal(counters.cpu().numpy(), o)
