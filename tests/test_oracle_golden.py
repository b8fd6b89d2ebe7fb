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
