"""Pin the CPU oracle against the reference: frozen known-answer values from
the reference's own tests and fixtures produced by running the reference
(tests/golden/make_golden.py). CPU only."""

import numpy as np
import pytest

from conftest import fixture_names, load_fixture, load_hashing

# the reference's own frozen goldens (tests/test_hashing.py:29-36, 56, 164-165)
FINALIZE_GOLDENS = {
    0x0000000000000000: 0x0000000000000000,
    0x0000000000000001: 0x5692161D100B05E5,
    0x0000000000000002: 0xDBD238973A2B148A,
    0x000000000000002A: 0xA759EA27D4727622,
    0x123456789ABCDEF0: 0x9629F58E8EC5B906,
    0xFFFFFFFFFFFFFFFF: 0xB4D055FCF2CBBD7B,
}


def test_oracle_finalize_known_answers(oracle):
    xs = np.array(list(FINALIZE_GOLDENS), dtype=np.uint64)
    assert [int(v) for v in oracle.mix_batch(xs)] == list(FINALIZE_GOLDENS.values())
    assert int(oracle.seed_array(0, 0, 1)[0]) == 0xE220A8397B1DCDAF


def test_oracle_key_from_string_known_answers(oracle):
    for s, want in {"apple": 0xBA8E799DCEB3BCB1, "": 0xF52A15E9A9B5E89B}.items():
        b = np.frombuffer(s.encode(), dtype=np.uint8).reshape(1, -1) if s else np.zeros((1, 0), np.uint8)
        assert int(oracle.keys_from_records(b)[0]) == want


def test_oracle_hashing_fixture(oracle):
    h = load_hashing()
    ins = np.array([int(x) for x in h["mix_batch_in"]], dtype=np.uint64)
    assert [str(int(v)) for v in oracle.mix_batch(ins)] == h["mix_batch_out"]
    for k, want in h["finalize"].items():
        assert int(oracle.mix_batch(np.array([int(k)], dtype=np.uint64))[0]) == int(want)
    for key, want in h["seeds"].items():
        m, d = (int(x) for x in key.split(":"))
        assert [str(int(s)) for s in oracle.seed_array(m, 0, d)] == want
    for key, want in h["seed_array_ext"].items():
        m, d = (int(x) for x in key.split(":"))
        assert [str(int(s)) for s in oracle.seed_array(m, d, d)] == want
    for s, want in h["key_from_string"].items():
        b = s.encode("utf-8")
        arr = np.frombuffer(b, dtype=np.uint8).reshape(1, -1) if b else np.zeros((1, 0), np.uint8)
        assert int(oracle.keys_from_records(arr)[0]) == int(want)


def replay_oracle(oracle, fx):
    kind = str(fx["kind"])
    sk = oracle.OracleSketch(kind, int(fx["d"]), int(fx["w"]), int(fx["z"]), int(fx["w_prime"]),
                             int(fx["master_seed"]))
    if "pre_fat" in fx:
        sk.fat[...] = fx["pre_fat"]
    sk.slim[...] = fx["pre_slim"]
    ops, keys = fx["ops"], fx["keys"].astype(np.uint64)
    bounds = np.linspace(0, len(ops), int(fx["batches"]) + 1).astype(int)
    status, idx = 0, -1
    for a, b in zip(bounds[:-1], bounds[1:]):
        st, oi, _ = sk.apply_ops(ops[a:b], keys[a:b])
        if st:
            status, idx = st, a + oi
            break
    return sk, status, idx


@pytest.mark.parametrize("name", fixture_names())
def test_oracle_matches_reference_fixture(oracle, name):
    fx = load_fixture(name)
    sk, status, idx = replay_oracle(oracle, fx)
    assert (status, idx) == (int(fx["status"]), int(fx["op_index"]))
    np.testing.assert_array_equal(sk.slim, fx["slim"])
    np.testing.assert_array_equal(sk.inc, fx["inc"])
    assert sk.seen == int(fx["seen"])
    if "fat" in fx:
        np.testing.assert_array_equal(sk.fat, fx["fat"])
    if "dsub" in fx:
        np.testing.assert_array_equal(sk.dsub, fx["dsub"])
    np.testing.assert_array_equal(sk.query_many(fx["query_keys"].astype(np.uint64)), fx["query"])
    np.testing.assert_array_equal(sk.query_many(fx["query_keys"].astype(np.uint64), threads=3), fx["query"])


def test_oracle_u32_keys_zero_extend(oracle):
    fx = load_fixture("sff_u32_medium")
    sk, _, _ = replay_oracle(oracle, fx)
    q32 = fx["query_keys"].astype(np.uint32)
    np.testing.assert_array_equal(sk.query_many(q32, threads=2), fx["query"])


# ---------------------------------------------------------------- Count / CML / oracle-assisted
from conftest import baseline_fixture_names, load_baseline_fixture  # noqa: E402


def _splits(n, batches):
    b = np.linspace(0, n, batches + 1).astype(int)
    return list(zip(b[:-1], b[1:]))


@pytest.mark.parametrize("name", baseline_fixture_names())
def test_oracle_matches_reference_baseline_fixture(oracle, name):
    """Count (_kernels.py:118-179), CML (_kernels.py:182-226, baselines.py:174-179)
    and the oracle-assisted slim (_kernels.py:387-411) against the reference's
    own outputs (tests/golden/make_golden_baselines.py)."""
    fx = load_baseline_fixture(name)
    kind, d, w = str(fx["kind"]), int(fx["d"]), int(fx["w"])
    seeds = oracle.seed_array(int(fx["master_seed"]), 0, d)
    keys = fx["keys"].astype(np.uint64)
    qk = fx["query_keys"].astype(np.uint64)
    status, idx, seen = 0, -1, 0
    if kind == "count":
        c = fx["pre_counters"].copy()
        for a, b in _splits(len(keys), int(fx["batches"])):
            st, oi, ni = oracle.count_apply(c, seeds, fx["ops"][a:b], keys[a:b])
            seen += ni
            if st:
                status, idx = st, a + oi
                break
        np.testing.assert_array_equal(c, fx["counters"])
        np.testing.assert_array_equal(oracle.count_query(c, seeds, qk), fx["query"])
        np.testing.assert_array_equal(oracle.count_query(c, seeds, qk), fx["collector_query"])
    elif kind == "cml":
        e = fx["pre_exponents"].copy()
        base, rs = float(fx["base"]), int(fx["rng_seed"])
        for a, b in _splits(len(keys), int(fx["batches"])):
            st, oi, ni = oracle.cml_apply(e, seeds, fx["ops"][a:b], keys[a:b], base, rs, seen)
            seen += ni
            if st:
                status, idx = st, a + oi
                break
        np.testing.assert_array_equal(e, fx["exponents"])
        with np.errstate(over="ignore", invalid="ignore"):
            np.testing.assert_array_equal(oracle.cml_value(oracle.cml_min_exp(e, seeds, qk), base), fx["query"])
    else:
        slim = fx["pre_slim"].copy()
        inc = np.zeros(d, np.int64)
        for a, b in _splits(len(keys), int(fx["batches"])):
            st, oi, ni = oracle.oracle_slim_apply(slim, seeds, keys[a:b], fx["true_counts"][a:b], inc)
            seen += ni
            if st:
                status, idx = st, a + oi
                break
        np.testing.assert_array_equal(slim, fx["slim"])
        np.testing.assert_array_equal(inc, fx["inc"])
        np.testing.assert_array_equal(oracle.min_query(slim, seeds, qk), fx["query"])
    assert (status, idx) == (int(fx["status"]), int(fx["op_index"]))
    assert seen == int(fx["seen"])
