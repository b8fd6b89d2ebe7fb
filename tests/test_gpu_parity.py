"""GPU parity: the CUDA path (parallel engine and the exact sequential device
engine) against the reference's golden fixtures and against the CPU oracle on
the BASELINE configurations. Bit-exact on every counter, tally and estimate."""

import numpy as np
import pytest
import torch

from conftest import fixture_names, load_fixture, load_hashing
from gpu_util import apply_batches, assert_state_equal, counters_of, host, make_sketch, set_state

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("parallel_engine_only")]

import paper_1701_04148_b200 as P  # noqa: E402
from paper_1701_04148_b200 import device as D  # noqa: E402
from paper_1701_04148_b200 import workloads as W  # noqa: E402


def test_device_hash_goldens():
    h = load_hashing()
    ins = np.array([int(x) for x in h["mix_batch_in"]], dtype=np.uint64)
    got = host(D.mix_batch(ins))
    assert [str(int(v)) for v in got] == h["mix_batch_out"]
    fin = np.array([int(k) for k in h["finalize"]], dtype=np.uint64)
    assert [int(v) for v in host(D.mix_batch(fin))] == [int(v) for v in h["finalize"].values()]
    for s, want in h["key_from_string"].items():
        b = s.encode("utf-8")
        if not b:
            continue
        rec = np.frombuffer(b, dtype=np.uint8).reshape(1, -1)
        assert int(host(D.load_keys(rec))[0]) == int(want)


@pytest.mark.parametrize("sequential", [False, True])
@pytest.mark.parametrize("name", fixture_names())
def test_fixture_parity(name, sequential):
    fx = load_fixture(name)
    kind = str(fx["kind"])
    sk = make_sketch(kind, int(fx["d"]), int(fx["w"]), int(fx["z"]), int(fx["w_prime"]), int(fx["master_seed"]))
    set_state(sk, fx)
    status, idx = apply_batches(sk, fx["ops"], fx["keys"], int(fx["batches"]), sequential)
    assert (status, idx) == (int(fx["status"]), int(fx["op_index"]))
    assert_state_equal(sk, fx["slim"], fx["inc"], fx["seen"], fx.get("fat"), fx.get("dsub"))
    np.testing.assert_array_equal(host(sk.query_many(fx["query_keys"])), fx["query"])
    assert P.export_slim(sk) == fx["export"].tobytes()


def oracle_run(oracle, kind, d, w, z, wp, seed, ops, keys_u64):
    o = oracle.OracleSketch(kind, d, w, z, wp, seed)
    r = o.apply_ops(ops, keys_u64)
    return o, r


def compare_cfg(oracle, kind, d, w, z, wp, seed, ops, keys, keys_u64, qkeys, qkeys_u64=None):
    o, (st, oi, _) = oracle_run(oracle, kind, d, w, z, wp, seed, ops, keys_u64)
    sk = make_sketch(kind, d, w, z, wp, seed)
    dev_ops = torch.from_numpy(ops).cuda()
    dev_keys = torch.from_numpy(keys).cuda() if isinstance(keys, np.ndarray) else keys
    status, idx = apply_batches(sk, dev_ops, dev_keys)
    assert (status, idx) == (st, oi)
    assert_state_equal(sk, o.slim, o.inc, o.seen, o.fat, o.dsub)
    if qkeys_u64 is None:
        qkeys_u64 = np.asarray(qkeys).astype(np.uint64)
    np.testing.assert_array_equal(host(sk.query_many(qkeys)), o.query_many(qkeys_u64))
    return sk


def test_cfg1_sf1_full(oracle):
    c = W.cfg1(seed=2017)
    compare_cfg(oracle, "sf1", 4, 16384, 4, 65536, 2017, c["ops"], c["keys"], c["keys"].astype(np.uint64),
                c["distinct"])


@pytest.mark.parametrize("kind", ["cm", "cu"])
def test_cfg2_full(oracle, kind):
    c = W.cfg2(seed=2017)
    compare_cfg(oracle, kind, 4, 65536, 1, None, 2017, c["ops"], c["keys"], c["keys"].astype(np.uint64),
                c["distinct"][:200000])


@pytest.mark.parametrize("alpha", [0.5, 1.0, 1.5])
def test_cfg3_sff_full(oracle, alpha):
    c = W.cfg3(seed=2017, alpha=alpha)
    sk = compare_cfg(oracle, "sff", 4, 65536, 4, None, 2017, c["ops"], c["keys"], c["keys"].astype(np.uint64),
                     c["distinct"])
    sk.check_invariants()


def test_cfg4_sf1_records(oracle):
    c = W.cfg4(seed=2017, n=20_000_000, v=2_000_000)
    keys_u64 = oracle.keys_from_records(c["records"])
    q = c["distinct"][:100000]
    compare_cfg(oracle, "sf1", 4, 12800, 1, 4194304, 2017, c["ops"], c["records"], keys_u64, q,
                oracle.keys_from_records(q))


def test_chunked_batches_equal_one_batch(oracle):
    c = W.cfg3(seed=7, n_ins=400_000, v=20_000, alpha=1.2)
    o, _ = oracle_run(oracle, "sff", 4, 4096, 4, None, 7, c["ops"], c["keys"].astype(np.uint64))
    sk = make_sketch("sff", 4, 4096, 4, None, 7)
    apply_batches(sk, c["ops"], c["keys"], batches=7)
    assert_state_equal(sk, o.slim, o.inc, o.seen, o.fat)


@pytest.mark.parametrize("kind", ["sff", "sf1", "cm", "cu"])
def test_prefix_semantics_at_scale(oracle, kind):
    """A failing op deep inside a large batch: the prefix is applied, the
    failing op leaves no trace (_kernels.py:4-8)."""
    c = W.cfg3(seed=3, n_ins=200_000, v=5000, alpha=1.0)
    ops, keys = c["ops"].copy(), c["keys"].copy()
    if kind in ("sf1", "cu"):
        ops = np.zeros_like(ops)
        ops[150_000] = 1  # unsupported delete
    else:
        keys[150_000] = np.uint32(0xDEADBEEF)  # never inserted
        ops[150_000] = 1  # phantom
    compare_cfg(oracle, kind, 4, 1024, 4, None, 3, ops, keys, keys.astype(np.uint64), c["distinct"])


def test_saturation_prefix_at_scale(oracle):
    c = W.cfg1(seed=4, n=100_000, v=300)
    for kind, z in (("sff", 4), ("sf1", 4)):
        o = oracle.OracleSketch(kind, 4, 64, z, None, 4)
        o.fat[...] = np.uint32(0xFFFFFFFF - 2000)
        st = o.apply_ops(c["ops"], c["keys"].astype(np.uint64))
        assert st[0] == 2
        sk = make_sketch(kind, 4, 64, z, None, 4)
        sk.fat.counters.fill_(0xFFFFFFFF - 2000)
        status, idx = apply_batches(sk, c["ops"], c["keys"])
        assert (status, idx) == st[:2]
        assert_state_equal(sk, o.slim, o.inc, o.seen, o.fat)


def long_run_stream(seed, w, n_bg, blocks, block_len, del_p):
    """Background traffic over many keys, interleaved with long blocks of one
    hot key's own inserts and deletes (every delete valid): the engine's
    multi-word runs, in and out of the steady regime."""
    rng = np.random.default_rng(seed)
    bg = rng.integers(1, 1 << 31, size=300, dtype=np.uint64).astype(np.uint32)
    ops, keys = [], []
    counts = {}
    for b in range(blocks):
        for _ in range(n_bg):  # background inserts (and deletes of inserted keys)
            k = int(bg[rng.integers(0, bg.size)])
            if counts.get(k, 0) and rng.random() < 0.3:
                ops.append(1); counts[k] -= 1
            else:
                ops.append(0); counts[k] = counts.get(k, 0) + 1
            keys.append(k)
        hot = int(bg[b % 7])
        for _ in range(block_len):
            if counts.get(hot, 0) and rng.random() < del_p:
                ops.append(1); counts[hot] -= 1
            else:
                ops.append(0); counts[hot] = counts.get(hot, 0) + 1
            keys.append(hot)
    return np.array(ops, np.uint8), np.array(keys, np.uint32)


@pytest.mark.parametrize("seed,w,del_p", [(1, 64, 0.3), (2, 256, 0.45), (3, 32, 0.49), (4, 1024, 0.2),
                                          (5, 16, 0.4)])
def test_sff_long_runs(oracle, seed, w, del_p):
    ops, keys = long_run_stream(seed, w, n_bg=400, blocks=12, block_len=3000, del_p=del_p)
    for sequential in (False, True):
        o, st = oracle_run(oracle, "sff", 4, w, 4, None, seed, ops, keys.astype(np.uint64))
        sk = make_sketch("sff", 4, w, 4, None, seed)
        status, idx = apply_batches(sk, ops, keys, sequential=sequential)
        assert (status, idx) == st[:2]
        assert_state_equal(sk, o.slim, o.inc, o.seen, o.fat)


@pytest.mark.parametrize("variant,wp", [("sf2", 16384), ("sf3", 16384), ("sf4", None)])
@pytest.mark.parametrize("alpha", [0.8, 1.2])
def test_sum_trigger_variants_at_scale(oracle, variant, wp, alpha):
    """SF2 / SF3 / SF4 on the parallel engine (bucket or fold-group sums, the
    deletion sub-sketch) against the oracle on a cfg-3 style stream."""
    c = W.cfg3(seed=5, n_ins=1_000_000, v=50_000, alpha=alpha)
    compare_cfg(oracle, variant, 4, 4096, 4, wp, 5, c["ops"], c["keys"], c["keys"].astype(np.uint64),
                c["distinct"])


@pytest.mark.parametrize("variant", ["sf2", "sf3", "sf4"])
@pytest.mark.parametrize("seed,w,del_p", [(1, 64, 0.3), (3, 32, 0.49), (5, 16, 0.4)])
def test_sum_trigger_long_runs(oracle, variant, seed, w, del_p):
    ops, keys = long_run_stream(seed, w, n_bg=400, blocks=12, block_len=3000, del_p=del_p)
    wp = 4 * w if variant in ("sf2", "sf3") else None
    for sequential in (False, True):
        o, st = oracle_run(oracle, variant, 4, w, 4, wp, seed, ops, keys.astype(np.uint64))
        sk = make_sketch(variant, 4, w, 4, wp, seed)
        status, idx = apply_batches(sk, ops, keys, sequential=sequential)
        assert (status, idx) == st[:2]
        assert_state_equal(sk, o.slim, o.inc, o.seen, o.fat, o.dsub)


@pytest.mark.parametrize("variant", ["sf2", "sf3", "sf4"])
def test_sum_trigger_prefix_semantics(oracle, variant):
    """A phantom delete deep inside a batch: the prefix applies, the failing
    op leaves no trace, on the parallel engine."""
    c = W.cfg3(seed=9, n_ins=200_000, v=5000, alpha=1.0)
    ops, keys = c["ops"].copy(), c["keys"].copy()
    keys[150_000] = np.uint32(0xDEADBEEF)
    ops[150_000] = 1
    wp = 4096 if variant in ("sf2", "sf3") else None
    compare_cfg(oracle, variant, 4, 1024, 4, wp, 9, ops, keys, keys.astype(np.uint64), c["distinct"])


@pytest.mark.parametrize("variant", ["sf2", "sf3", "sf4", "sff"])
@pytest.mark.parametrize("d,w,z", [(1, 97, 2), (2, 64, 1), (3, 50, 8), (8, 33, 3), (4, 1000, 5)])
def test_deleting_variants_shapes(oracle, variant, d, w, z):
    """Every deleting variant on the parallel engine across d, odd widths and
    slot counts (z up to 8), against the oracle and the sequential engine."""
    rng = np.random.default_rng(d * 131 + w * 7 + z)
    distinct = rng.integers(0, 1 << 32, size=300, dtype=np.uint64).astype(np.uint32)
    ops, keys, counts = [], [], {}
    for _ in range(40_000):
        k = int(distinct[min(int(rng.zipf(1.3)) - 1, distinct.size - 1)])
        if counts.get(k, 0) and rng.random() < 0.35:
            ops.append(1); counts[k] -= 1
        else:
            ops.append(0); counts[k] = counts.get(k, 0) + 1
        keys.append(k)
    ops, keys = np.array(ops, np.uint8), np.array(keys, np.uint32)
    wp = z * w if variant in ("sf2", "sf3") else None
    o, st = oracle_run(oracle, variant, d, w, z, wp, d + z, ops, keys.astype(np.uint64))
    for sequential in (False, True):
        sk = make_sketch(variant, d, w, z, wp, d + z)
        status, idx = apply_batches(sk, ops, keys, batches=3, sequential=sequential)
        assert (status, idx) == st[:2]
        assert_state_equal(sk, o.slim, o.inc, o.seen, o.fat, o.dsub)


@pytest.mark.parametrize("d,w,wp,batches", [(4, 64, 256, 1), (4, 128, 4096, 3), (2, 32, 64, 2), (8, 200, 1000, 1),
                                            (4, 12800, 4194304, 1)])
def test_sf1_dropped_pairs(oracle, d, w, wp, batches):
    """SF1 drops (op, row >= 1) pairs whose cell provably exceeds the op's
    b_min (a hot key's count on the cell). Hot keys mixed with many cold keys
    on narrow rows make such pairs common; state must stay bit-exact, across
    batches, against the oracle and the sequential engine."""
    rng = np.random.default_rng(d * 7 + w + batches)
    hot = rng.integers(0, 1 << 32, size=5, dtype=np.uint64).astype(np.uint32)
    cold = rng.integers(0, 1 << 32, size=20000, dtype=np.uint64).astype(np.uint32)
    n = 200_000
    pick_hot = rng.random(n) < 0.5
    keys = np.where(pick_hot, hot[rng.integers(0, hot.size, n)], cold[rng.integers(0, cold.size, n)]).astype(np.uint32)
    ops = np.zeros(n, np.uint8)
    o, st = oracle_run(oracle, "sf1", d, w, 1, wp, 3, ops, keys.astype(np.uint64))
    for sequential in (False, True):
        sk = make_sketch("sf1", d, w, 1, wp, 3)
        status, idx = apply_batches(sk, ops, keys, batches=batches, sequential=sequential)
        assert (status, idx) == st[:2]
        assert_state_equal(sk, o.slim, o.inc, o.seen, o.fat)


@pytest.mark.parametrize("kind", ["sf1", "cu"])
@pytest.mark.parametrize("d,w,preset", [(4, 64, "zero"), (4, 256, "random"), (3, 50, "skewed"), (8, 128, "random")])
def test_dropped_pairs_any_start_state(oracle, kind, d, w, preset):
    """The drop rules of SF1 (lower bound >= b_min) and CU (lower bound >
    upper bound of the op's minimum, from the cells' values before the batch)
    hold from any starting state: preset slim / fat counters, hot keys over
    narrow rows, several batches, every row droppable (row 0 included)."""
    rng = np.random.default_rng(d * 100 + w + len(preset))
    hot = rng.integers(0, 1 << 32, size=4, dtype=np.uint64).astype(np.uint32)
    cold = rng.integers(0, 1 << 32, size=5000, dtype=np.uint64).astype(np.uint32)
    n = 120_000
    keys = np.where(rng.random(n) < 0.4, hot[rng.integers(0, hot.size, n)],
                    cold[rng.integers(0, cold.size, n)]).astype(np.uint32)
    ops = np.zeros(n, np.uint8)
    wp = 4 * w if kind == "sf1" else None
    o = oracle.OracleSketch(kind, d, w, 1, wp, 5)
    if preset == "random":
        o.slim[...] = rng.integers(0, 3000, size=o.slim.shape).astype(np.uint32)
    elif preset == "skewed":
        o.slim[...] = (rng.pareto(1.2, size=o.slim.shape) * 50).astype(np.uint32)
    if o.fat is not None and preset != "zero":
        o.fat[...] = rng.integers(0, 2000, size=o.fat.shape).astype(np.uint32)
    sk = make_sketch(kind, d, w, 1, wp, 5)
    counters_of(sk).copy_(torch.from_numpy(o.slim.copy()))
    if o.fat is not None:
        sk.fat.counters.copy_(torch.from_numpy(o.fat.copy()))
    bounds = np.linspace(0, n, 4).astype(int)
    for a, b in zip(bounds[:-1], bounds[1:]):
        st = o.apply_ops(ops[a:b], keys[a:b].astype(np.uint64))
        assert st[0] == 0
        sk.apply_ops(ops[a:b], keys[a:b])
    assert_state_equal(sk, o.slim, o.inc, o.seen, o.fat)
