"""Synthetic generators (CPU): determinism and the structural promises of
SURVEY.md §8(d) at reduced sizes."""

import numpy as np

from paper_1701_04148_b200 import workloads as W


def test_cfg1_deterministic_and_shaped():
    a = W.cfg1(seed=5, n=20000, v=1000)
    b = W.cfg1(seed=5, n=20000, v=1000)
    np.testing.assert_array_equal(a["keys"], b["keys"])
    assert a["keys"].dtype == np.uint32 and a["ops"].sum() == 0
    assert np.unique(a["distinct"]).size == 1000
    assert set(np.unique(a["keys"])) <= set(a["distinct"])


def test_cfg3_deletes_follow_their_insert():
    c = W.cfg3(seed=9, n_ins=20000, v=500, alpha=1.0)
    ops, keys = c["ops"], c["keys"]
    assert int(ops.sum()) == 4000 and ops.size == 24000
    # running count per key never goes negative: every delete follows its insert
    cnt = {}
    for op, k in zip(ops.tolist(), keys.tolist()):
        cnt[k] = cnt.get(k, 0) + (1 if op == 0 else -1)
        assert cnt[k] >= 0


def test_cfg4_records():
    c = W.cfg4(seed=3, n=5000, v=300)
    assert c["records"].shape == (5000, 13) and c["records"].dtype == np.uint8


def test_query_keys_slices_and_presence():
    present = W.distinct_u32(W.rng_for(1), 2000)
    full = W.query_keys(11, present, 1.0, 0, 20000)
    np.testing.assert_array_equal(full[5000:7000], W.query_keys(11, present, 1.0, 5000, 7000))
    inset = np.isin(full, present)
    assert 0.45 < inset.mean() < 0.55
    uni = W.query_keys(11, present, 0.0, 0, 20000)
    assert 0.45 < np.isin(uni, present).mean() < 0.55
