"""Randomised differential test: every update engine against the CPU oracle
over random shapes (d 1..8, power-of-two and odd widths, z 1..8), random
key skews, delete mixes that include never-inserted keys (phantoms), preset
counter states near saturation, and several batches per stream."""

import os

import numpy as np
import pytest
import torch

from gpu_util import apply_batches, assert_state_equal, host, make_sketch

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("parallel_engine_only")]

KINDS = ["sff", "sf4", "sf3", "sf2", "sf1", "cm", "cu"]
# SFK_FUZZ_SEEDS scales every fuzz test (default 40 seeds each)
SEEDS = int(os.environ.get("SFK_FUZZ_SEEDS", "40"))
SEED0 = int(os.environ.get("SFK_FUZZ_SEED0", "0"))  # first seed; soak runs set it to explore new seeds


def random_case(rng, kind):
    d = int(rng.integers(1, 9))
    w = int(rng.choice([8, 16, 33, 64, 100, 256, 1000]))
    z = int(rng.integers(1, 9)) if kind in ("sff", "sf4", "sf3") else 1
    wp = None
    if kind in ("sf1", "sf2"):
        wp = int(w * rng.integers(1, 5) + rng.integers(0, 7))
    if kind == "sf3":
        wp = z * w
    v = int(rng.integers(5, 3000))
    n = int(rng.integers(1, 40_000))
    alpha = float(rng.uniform(0.0, 1.6))
    ranks = np.minimum(np.nan_to_num(rng.pareto(alpha + 0.05, size=n) * 3, posinf=v), v - 1).astype(np.int64)
    distinct = rng.integers(0, 1 << 40, size=v, dtype=np.uint64)
    keys = distinct[ranks]
    if kind in ("sf1", "cu"):
        ops = np.zeros(n, np.uint8)
        if rng.random() < 0.3:
            ops[int(rng.integers(0, n))] = 1  # an unsupported delete somewhere
    else:
        ops = (rng.random(n) < rng.uniform(0.0, 0.45)).astype(np.uint8)
        # deletes mostly of keys inserted before; some of never-seen keys
        strange = (ops == 1) & (rng.random(n) < 0.02)
        keys = np.where(strange, rng.integers(0, 1 << 40, size=n, dtype=np.uint64), keys)
    return d, w, z, wp, keys, ops


@pytest.mark.parametrize("sequential", [False, True])
@pytest.mark.parametrize("seed", range(SEED0, SEED0 + SEEDS))
@pytest.mark.parametrize("kind", KINDS)
def test_fuzz_against_oracle(oracle, kind, seed, sequential):
    if sequential and seed % 4:
        pytest.skip("the one-thread engine is fuzzed on every 4th seed")
    rng = np.random.default_rng(1000 * KINDS.index(kind) + seed)
    d, w, z, wp, keys, ops = random_case(rng, kind)
    o = oracle.OracleSketch(kind, d, w, z, wp, seed)
    sk = make_sketch(kind, d, w, z, wp, seed)
    if rng.random() < 0.3:  # preset state: counters near the top
        hi = np.uint32(0xFFFFFFFF - int(rng.integers(0, 40)))
        if o.fat is not None and rng.random() < 0.5:
            o.fat[...] = hi
            sk.fat.counters.copy_(torch.from_numpy(o.fat.copy()))
        elif kind in ("cm", "cu"):
            o.slim[...] = hi
            sk.counters.copy_(torch.from_numpy(o.slim.copy()))
    batches = int(rng.integers(1, 4))
    bounds = np.linspace(0, len(ops), batches + 1).astype(int)
    want = (0, -1)
    for a, b in zip(bounds[:-1], bounds[1:]):
        st, oi, _ = o.apply_ops(ops[a:b], keys[a:b])
        if st:
            want = (st, a + oi)
            break
    got = apply_batches(sk, ops, keys, batches=batches, sequential=sequential)
    assert got == want
    assert_state_equal(sk, o.slim, o.inc, o.seen, o.fat, o.dsub)
    q = np.unique(keys)[:2000]
    np.testing.assert_array_equal(host(sk.query_many(q)), o.query_many(q))


@pytest.mark.parametrize("seed", range(SEED0, SEED0 + SEEDS))
def test_fuzz_count_cml_oracle(oracle, seed):
    """Count, CML and the oracle-assisted slim over random shapes, presets
    (near the int32 / u16 / u32 bounds), bases, counts and batch splits."""
    import paper_1701_04148_b200 as P

    rng = np.random.default_rng(77_000 + seed)
    d = int(rng.integers(1, 11))
    w = int(rng.choice([8, 31, 64, 200, 1024]))
    n = int(rng.integers(1, 30_000))
    v = int(rng.integers(3, 2000))
    keys = rng.integers(0, 1 << 40, size=v, dtype=np.uint64)[rng.integers(0, v, size=n)]
    seeds = oracle.seed_array(seed, 0, d)
    batches = int(rng.integers(1, 4))
    bounds = np.linspace(0, n, batches + 1).astype(int)

    def run(apply_o, apply_g):
        want = (0, -1)
        for a, b in zip(bounds[:-1], bounds[1:]):
            st, oi, _ = apply_o(a, b)
            if st:
                want = (st, a + oi)
                break
        got = (0, -1)
        for a, b in zip(bounds[:-1], bounds[1:]):
            try:
                apply_g(a, b)
            except (P.SaturationError, P.UnsupportedOperationError, P.PhantomDeletionError) as e:
                got = ({P.PhantomDeletionError: 1, P.SaturationError: 2, P.UnsupportedOperationError: 3}[type(e)],
                       a + int(str(e).split(":")[0].split()[1]))
                break
        assert got == want

    # Count
    ops = (rng.random(n) < 0.3).astype(np.uint8)
    c = np.zeros((d, w), np.int32)
    if rng.random() < 0.4:
        c[...] = rng.choice(np.array([2147483647 - 3, -2147483648 + 3, 0], np.int32), size=c.shape)
    cs = P.CountSketch(P.SketchParams(d=d, w=w, master_seed=seed))
    cs.counters.copy_(torch.from_numpy(c.copy()))
    run(lambda a, b: oracle.count_apply(c, seeds, ops[a:b], keys[a:b]), lambda a, b: cs.apply_ops(ops[a:b], keys[a:b]))
    np.testing.assert_array_equal(host(cs.counters), c)
    np.testing.assert_array_equal(host(cs.query_many(keys[:500])), oracle.count_query(c, seeds, keys[:500]))
    # CML
    base = float(rng.choice([1.0001, 1.01, 1.08, 1.5, 3.0]))
    ops_c = np.zeros(n, np.uint8)
    if rng.random() < 0.2:
        ops_c[int(rng.integers(0, n))] = 1
    e = np.zeros((d, w), np.uint16)
    if rng.random() < 0.4:
        e[...] = rng.integers(0xFFF0, 0x10000, size=e.shape).astype(np.uint16)
    ml = P.CmlSketch(P.SketchParams(d=d, w=w, master_seed=seed), base=base, rng_seed=seed * 3)
    ml.exponents.copy_(torch.from_numpy(e.copy()))
    seen = [0]

    def cml_o(a, b):
        r = oracle.cml_apply(e, seeds, ops_c[a:b], keys[a:b], base, seed * 3, seen[0])
        seen[0] += r[2]
        return r

    run(cml_o, lambda a, b: ml.apply_ops(ops_c[a:b], keys[a:b]))
    np.testing.assert_array_equal(host(ml.exponents), e)
    assert ml.insertions_seen == seen[0]
    # oracle-assisted
    tc = rng.integers(-3, 40, size=n).astype(np.int64)
    if rng.random() < 0.2:
        tc[rng.integers(0, n, size=5)] = 1 << 40
    slim = np.zeros((d, w), np.uint32)
    if rng.random() < 0.3:
        slim[...] = np.uint32(0xFFFFFFFF - int(rng.integers(0, 30)))
    inc = np.zeros(d, np.int64)
    sk = P.SfSketch(P.SketchParams(d=d, w=w, z=2, master_seed=seed), "sff")
    sk.slim.counters.copy_(torch.from_numpy(slim.copy()))
    run(lambda a, b: oracle.oracle_slim_apply(slim, seeds, keys[a:b], tc[a:b], inc),
        lambda a, b: sk.oracle_assisted_apply(keys[a:b], tc[a:b]))
    np.testing.assert_array_equal(host(sk.slim.counters), slim)
    np.testing.assert_array_equal(host(sk.slim.increment_counts), inc)


@pytest.mark.parametrize("seed", range(SEED0, SEED0 + SEEDS))
def test_fuzz_query_paths(oracle, seed):
    """min_query over random shapes, value distributions (small, around the
    u16 code boundary 0xF800, up to 2^32 - 1), key kinds and every path the
    shape allows (auto, L2, shared memory, cluster, warp-pipelined cluster)."""
    import ctypes

    from paper_1701_04148_b200 import _lib

    rng = np.random.default_rng(55_000 + seed)
    d = int(rng.integers(1, 9))
    w = int(rng.choice([1, 7, 1000, 12800, 40000, 65536, 100_003, 1 << 18]))
    dist = rng.integers(0, 4)
    if dist == 0:
        c = rng.integers(0, 300, size=(d, w), dtype=np.uint64)
    elif dist == 1:
        c = rng.integers(0xF700, 0xF900, size=(d, w), dtype=np.uint64)
    elif dist == 2:
        c = rng.integers(0, 1 << 32, size=(d, w), dtype=np.uint64)
    else:
        c = np.where(rng.random((d, w)) < 0.01, rng.integers(60000, 1 << 32, size=(d, w), dtype=np.uint64),
                     rng.integers(0, 2000, size=(d, w), dtype=np.uint64))
    c = c.astype(np.uint32)
    n = int(rng.choice([1, 33, 5000, 300_000, 2_500_000]))
    kind = int(rng.integers(0, 3))
    seeds = oracle.seed_array(seed, 0, d)
    if kind == _lib.KEY_U32:
        keys = rng.integers(0, 1 << 32, size=n, dtype=np.uint64).astype(np.uint32)
        ku = keys.astype(np.uint64)
        kt, rec = torch.from_numpy(keys).cuda(), 0
    elif kind == _lib.KEY_U64:
        ku = rng.integers(0, np.iinfo(np.uint64).max, size=n, dtype=np.uint64)
        kt, rec = torch.from_numpy(ku).cuda(), 0
    else:
        rec = int(rng.integers(1, 20))
        recs = rng.integers(0, 256, size=(n, rec), dtype=np.uint8)
        ku = oracle.keys_from_records(recs)
        kt = torch.from_numpy(recs.reshape(-1)).cuda()
    want = oracle.min_query(c, seeds, ku, threads=4)
    ct = torch.from_numpy(c).cuda()
    L = _lib.lib()
    paths = [0, 1]
    if w * d * 4 <= 200 * 1024:
        paths.append(2)
    if 2 <= d <= 8 and w * 2 <= 110 * 1024:
        paths += [3, 4]
    for path in paths:
        prev = L.sfk_query_path(path)
        try:
            out = torch.full((n,), -1, dtype=torch.int64, device="cuda")
            _lib.check(L.sfk_min_query(ct.data_ptr(), seeds.ctypes.data_as(ctypes.c_void_p), d, w, kt.data_ptr(), kind,
                                       rec, n, out.data_ptr(), _lib.stream_ptr()), "sfk_min_query")
            torch.cuda.synchronize()
        finally:
            L.sfk_query_path(prev)
        np.testing.assert_array_equal(out.cpu().numpy(), want, err_msg=f"path {path}")
