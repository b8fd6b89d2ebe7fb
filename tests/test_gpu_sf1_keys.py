"""SF1 and CU on the parallel pipeline with the key grouping of round 2
(DESIGN.md §3.2a): 64-bit keys are grouped by the slot an open-addressing
table gives them, record keys are hashed once and read back as u64, and run
heads come from per-op break bits. These cases aim at that machinery: the
key 2^64 - 1 (the table's empty mark, which gets its own group id), keys
that differ only in high bits, tiny tables (heavy slot collisions in the
table's probe sequences), record keys, and a failing op in the middle of the
batch. Each is compared with the CPU oracle (`_kernels.py:91-115, 244-315`)."""

import numpy as np
import pytest
import torch

import paper_1701_04148_b200 as P
from gpu_util import apply_batches, assert_state_equal, host, make_sketch

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("parallel_engine_only")]

EMPTY = np.uint64(0xFFFFFFFFFFFFFFFF)


def _stream(rng, n, v, special):
    distinct = rng.integers(0, 1 << 63, size=v, dtype=np.uint64)
    distinct[: len(special)] = special
    ranks = np.minimum((rng.pareto(0.8, size=n) * 2).astype(np.int64), v - 1)
    return distinct[ranks]


@pytest.mark.parametrize("kind", ["sf1", "cu"])
@pytest.mark.parametrize("seed", range(6))
def test_u64_keys_with_the_empty_mark(oracle, kind, seed):
    rng = np.random.default_rng(700 + seed)
    special = np.array([EMPTY, EMPTY - np.uint64(1), np.uint64(0), np.uint64(1 << 63), np.uint64((1 << 63) | 1)],
                       dtype=np.uint64)
    n = int(rng.integers(20_000, 120_000))
    keys = _stream(rng, n, int(rng.integers(50, 5000)), special)
    keys[rng.integers(0, n, size=200)] = EMPTY  # the mark itself, often
    ops = np.zeros(n, np.uint8)
    if seed % 2:
        ops[int(rng.integers(n // 4, n))] = 1  # SF1 / CU: a delete is the failing op
    d, w = 4, int(rng.choice([64, 100, 1024]))
    wp = 4 * w + 3 if kind == "sf1" else None
    o = oracle.OracleSketch(kind, d, w, 1, wp, seed)
    st, oi, _ = o.apply_ops(ops, keys)
    sk = make_sketch(kind, d, w, 1, wp, seed)
    got = apply_batches(sk, ops, keys)
    assert got == ((st, oi) if st else (0, -1))
    assert_state_equal(sk, o.slim, o.inc, o.seen, o.fat if kind == "sf1" else None)
    q = np.unique(keys)
    np.testing.assert_array_equal(host(sk.query_many(q)), o.query_many(q))


@pytest.mark.parametrize("seed", range(4))
def test_sf1_record_keys_midsize(oracle, seed):
    """13-B records: hashed once into u64 (FNV-1a + finalize64,
    `hashing.py:124-129`), then grouped through the slot table."""
    rng = np.random.default_rng(800 + seed)
    v, n = int(rng.integers(100, 20_000)), int(rng.integers(50_000, 400_000))
    recs = rng.integers(0, 256, size=(v, 13), dtype=np.uint8)
    ranks = np.minimum((rng.pareto(1.0, size=n) * 3).astype(np.int64), v - 1)
    records = np.ascontiguousarray(recs[ranks])
    ops = np.zeros(n, np.uint8)
    params = P.SketchParams(d=4, w=1280, w_prime=16384 + seed, master_seed=seed)
    sk = P.SfSketch(params, "sf1")
    sk.apply_ops(torch.from_numpy(ops).cuda(), torch.from_numpy(records).cuda())
    keys = oracle.keys_from_records(records)
    o = oracle.OracleSketch("sf1", 4, 1280, 1, 16384 + seed, seed)
    assert o.apply_ops(ops, keys)[0] == 0
    assert_state_equal(sk, o.slim, o.inc, o.seen, o.fat)


@pytest.fixture
def shared_cell_fat_path(monkeypatch):
    """Route every SF1 batch through the shared-cell fat phase (normally
    batches of >= 2^20 ops only; DESIGN.md §8 item 3)."""
    monkeypatch.setenv("SFK_SF1_FAT_MIN", "1")
    yield


@pytest.mark.usefixtures("shared_cell_fat_path")
@pytest.mark.parametrize("seed", range(40))
def test_sf1_shared_cell_fat_phase(oracle, seed):
    """Random shapes (tiny fat widths: most cells shared; wide ones: most
    exclusive), warm sketches, saturation presets on the fat and mid-batch
    deletes (both fall back to the full sort), several batches."""
    rng = np.random.default_rng(900 + seed)
    d = int(rng.integers(2, 9))
    w = int(rng.choice([16, 100, 1024]))
    wp = int(rng.choice([w, 4 * w + 1, 64 * w + 7]))
    v, n = int(rng.integers(5, 5000)), int(rng.integers(100, 60_000))
    keys = _stream(rng, n, v, np.array([EMPTY], dtype=np.uint64))
    ops = np.zeros(n, np.uint8)
    if rng.random() < 0.25:
        ops[int(rng.integers(0, n))] = 1
    o = oracle.OracleSketch("sf1", d, w, 1, wp, seed)
    sk = make_sketch("sf1", d, w, 1, wp, seed)
    r = rng.random()
    if r < 0.2:  # near saturation
        o.fat[...] = np.uint32(0xFFFFFFFF - int(rng.integers(0, 60)))
        sk.fat.counters.copy_(torch.from_numpy(o.fat.copy()))
    elif r < 0.5:  # warm: fat and slim from an earlier batch
        pre = _stream(rng, 5000, v, np.array([], dtype=np.uint64))
        o.apply_ops(np.zeros(pre.size, np.uint8), pre)
        sk.apply_ops(np.zeros(pre.size, np.uint8), pre)
    batches = int(rng.integers(1, 3))
    bounds = np.linspace(0, n, batches + 1).astype(int)
    want = (0, -1)
    for a, b in zip(bounds[:-1], bounds[1:]):
        st, oi, _ = o.apply_ops(ops[a:b], keys[a:b])
        if st:
            want = (st, a + oi)
            break
    got = apply_batches(sk, ops, keys, batches=batches)
    assert got == want
    assert_state_equal(sk, o.slim, o.inc, o.seen, o.fat)
