"""GPU tests of the drop-in API surface: the reference's pinned
micro-scenarios (tests/test_sf.py, test_baselines.py, test_serialize.py of the
reference restated), error semantics, edge shapes (empty batches, d = 1 / 8 /
9, z = 1 / 8, non-power-of-two widths, 64-bit / 32-bit / record keys), the
export -> import -> collector round trip and the oracle-assisted mode, each
checked against the CPU oracle."""

import numpy as np
import pytest
import torch

from gpu_util import apply_batches, assert_state_equal, host, make_sketch

pytestmark = pytest.mark.gpu

import paper_1701_04148_b200 as P  # noqa: E402
from paper_1701_04148_b200 import workloads as W  # noqa: E402
from paper_1701_04148_b200.hashing import bucket_hash, derive_seeds, slot_hash  # noqa: E402

ALL = ("sf1", "sf2", "sf3", "sf4", "sff")
DELETING = ("sf2", "sf3", "sf4", "sff")


@pytest.mark.parametrize("variant", ALL)
def test_first_insert_sets_all_slim_counters(variant):
    s = P.SfSketch(P.SketchParams(d=3, w=8, z=2), variant)
    s.insert(42)
    assert int(s.slim.counters.to(torch.int64).sum()) == 3
    assert s.query(42) == 1 and s.query(7) == 0


@pytest.mark.parametrize("variant", ALL)
def test_single_item_counts_exactly(variant):
    s = P.SfSketch(P.SketchParams(d=2, w=4, z=2), variant)
    for _ in range(9):
        s.insert(123)
    assert s.query(123) == 9


@pytest.mark.parametrize("variant", DELETING)
def test_insert_then_delete_returns_to_zero(variant):
    s = P.SfSketch(P.SketchParams(d=3, w=16, z=2), variant)
    s.insert(77)
    s.delete(77)
    assert s.query(77) == 0
    assert int(s.fat.counters.to(torch.int64).sum()) == 0


def test_second_insert_skips_non_minimal_shared_counter():
    d, w, z = 2, 8, 16
    fam = derive_seeds(0, d)
    e1 = 1
    b1 = [bucket_hash(fam, i, e1, w) for i in range(d)]
    e2 = next(c for c in range(2, 50000)
              if bucket_hash(fam, 0, c, w) == b1[0] and bucket_hash(fam, 1, c, w) != b1[1]
              and slot_hash(fam, 0, c, z) != slot_hash(fam, 0, e1, z))
    s = P.SfSketch(P.SketchParams(d=d, w=w, z=z), "sff")
    s.insert(e1)
    s.insert(e2)
    sl = host(s.slim.counters)
    assert sl[0, b1[0]] == 1 and s.query(e1) == 1 and s.query(e2) == 1


def test_error_semantics():
    s = P.SfSketch(P.SketchParams(d=2, w=4), "sf1")
    s.insert(5)
    with pytest.raises(P.UnsupportedOperationError):
        s.delete(5)
    for v in DELETING:
        with pytest.raises(P.PhantomDeletionError):
            P.SfSketch(P.SketchParams(d=2, w=4, z=2), v).delete(5)
    t = P.SfSketch(P.SketchParams(d=2, w=4, z=2), "sff")
    t.fat.counters.fill_(0xFFFFFFFF)
    with pytest.raises(P.SaturationError):
        t.insert(1)
    with pytest.raises(P.ConfigurationError):
        P.SfSketch(P.SketchParams(d=2, w=4, z=2, w_prime=9), "sf3")
    with pytest.raises(P.ConfigurationError):
        s.apply_ops(np.array([0, 2], np.uint8), np.array([1, 2], np.uint64))
    with pytest.raises(P.ConfigurationError):
        s.apply_ops(np.array([0], np.uint8), np.array([1, 2], np.uint64))
    with pytest.raises(P.UnsupportedOperationError):
        P.CuSketch(P.SketchParams(d=2, w=4)).delete(3)


def test_prefix_applied_and_seen_counted_on_abort(oracle):
    ops = np.array([0, 0, 0, 1, 0], np.uint8)
    keys = np.array([1, 2, 3, 99, 4], np.uint64)
    s = P.SfSketch(P.SketchParams(d=2, w=8, z=2, master_seed=3), "sff")
    with pytest.raises(P.PhantomDeletionError) as ei:
        s.apply_ops(ops, keys)
    assert "op 3" in str(ei.value) and "99" in str(ei.value)
    assert s.slim.insertions_seen == 3
    o = oracle.OracleSketch("sff", 2, 8, 2, None, 3)
    o.apply_ops(ops, keys)
    assert_state_equal(s, o.slim, o.inc, o.seen, o.fat)


@pytest.mark.parametrize("kind", ["sff", "sf1", "cm", "cu", "sf4", "sf2", "sf3"])
def test_empty_batch(kind):
    sk = make_sketch(kind, 2, 8, 2, None, 0)
    sk.apply_ops(np.zeros(0, np.uint8), np.zeros(0, np.uint64))
    assert host(sk.query_many(np.zeros(0, np.uint64))).shape == (0,)


@pytest.mark.parametrize("kind,d,w,z,wp", [
    ("sff", 1, 64, 1, None), ("sff", 8, 128, 8, None), ("sff", 9, 32, 3, None), ("sff", 4, 100, 5, None),
    ("sf1", 1, 37, 1, 91), ("sf1", 8, 64, 2, None), ("sf1", 9, 32, 1, 1000), ("sf1", 4, 12800, 1, 4194304),
    ("cu", 8, 50, 1, None), ("cm", 9, 33, 1, None), ("cu", 1, 7, 1, None), ("cm", 3, 65536, 1, None),
])
def test_shapes_against_oracle(oracle, kind, d, w, z, wp):
    c = W.cfg3(seed=d * 7 + w, n_ins=30_000, v=800, alpha=1.1)
    ops, keys = c["ops"], c["keys"]
    if kind in ("sf1", "cu"):
        ops = np.zeros_like(ops)
    o = oracle.OracleSketch(kind, d, w, z, wp, 11)
    st = o.apply_ops(ops, keys.astype(np.uint64))
    sk = make_sketch(kind, d, w, z, wp, 11)
    assert apply_batches(sk, ops, keys) == st[:2]
    assert_state_equal(sk, o.slim, o.inc, o.seen, o.fat)
    np.testing.assert_array_equal(host(sk.query_many(c["distinct"])), o.query_many(c["distinct"].astype(np.uint64)))


def test_key_dtypes_agree():
    rng = np.random.Generator(np.random.PCG64(1))
    k32 = rng.integers(0, 1 << 32, size=5000, dtype=np.uint64).astype(np.uint32)
    res = []
    for keys in (k32, k32.astype(np.uint64), k32.astype(np.int64), torch.from_numpy(k32).cuda(), list(map(int, k32))):
        s = P.SfSketch(P.SketchParams(d=4, w=256, z=4, master_seed=9), "sff")
        s.apply_ops(np.zeros(len(k32), np.uint8), keys)
        res.append(host(s.slim.counters))
    for r in res[1:]:
        np.testing.assert_array_equal(res[0], r)
    big = np.array([2**64 - 1, 2**63, 0], np.uint64)
    s = P.CmSketch(P.SketchParams(d=3, w=16))
    s.apply_ops(np.zeros(3, np.uint8), big)
    assert [s.query(int(k)) for k in big] == [1, 1, 1]


def test_record_keys_match_key_from_string(oracle):
    recs = np.frombuffer(b"flow:10.0.0.1" b"flow:10.0.0.2" b"flow:10.0.0.1", dtype=np.uint8).reshape(3, 13)
    s = P.SfSketch(P.SketchParams(d=4, w=64, w_prime=1000, master_seed=2), "sf1")
    s.apply_ops(np.zeros(3, np.uint8), recs)
    assert s.query(P.key_from_string("flow:10.0.0.1")) == 2
    assert s.query(P.key_from_string("flow:10.0.0.2")) == 1
    assert host(s.query_many(recs)).tolist() == [2, 1, 2]


def test_export_import_collector_roundtrip():
    c = W.cfg3(seed=3, n_ins=50_000, v=2000)
    s = P.SfSketch(P.SketchParams(d=4, w=512, z=4, master_seed=77), "sff")
    s.apply_ops(c["ops"], c["keys"])
    payload = s.export_slim()
    col = P.import_slim(payload)
    assert col.export() == payload and col.insertions_seen == 50_000 and col.variant_code == 6
    np.testing.assert_array_equal(host(col.query_many(c["distinct"])), host(s.query_many(c["distinct"])))
    for cls in (P.CmSketch, P.CuSketch):
        b = cls(P.SketchParams(d=3, w=64, master_seed=5))
        b.apply_ops(np.zeros(1000, np.uint8), c["keys"][:1000])
        bc = P.import_slim(P.export_slim(b))
        np.testing.assert_array_equal(host(bc.query_many(c["distinct"][:100])), host(b.query_many(c["distinct"][:100])))


def test_oracle_assisted_mode(oracle):
    keys = np.array([5, 5, 6, 5, 7, 6], np.uint64)
    true = np.array([1, 2, 1, 3, 1, 2], np.int64)
    s = P.SfSketch(P.SketchParams(d=3, w=8, z=2, master_seed=1), "sff")
    s.oracle_assisted_apply(keys, true)
    slim = np.zeros((3, 8), np.uint32)
    inc = np.zeros(3, np.int64)
    oracle.oracle_slim_apply(slim, oracle.seed_array(1, 0, 3), keys, true, inc)
    np.testing.assert_array_equal(host(s.slim.counters), slim)
    with pytest.raises(P.UnsupportedOperationError):
        s.insert(3)


def test_invariants_hold_after_mixed_stream():
    c = W.cfg3(seed=8, n_ins=100_000, v=3000, alpha=1.3)
    for v in ("sff", "sf4"):
        s = P.SfSketch(P.SketchParams(d=4, w=256, z=4, master_seed=8), v)
        s.apply_ops(c["ops"], c["keys"])
        s.check_invariants()


def test_parallel_equals_sequential_engine():
    c = W.cfg3(seed=12, n_ins=200_000, v=4000, alpha=1.2)
    a = P.SfSketch(P.SketchParams(d=4, w=1024, z=4, master_seed=12), "sff")
    b = P.SfSketch(P.SketchParams(d=4, w=1024, z=4, master_seed=12), "sff")
    a.apply_ops(c["ops"], c["keys"])
    b.apply_ops(c["ops"], c["keys"], sequential=True)
    np.testing.assert_array_equal(host(a.slim.counters), host(b.slim.counters))
    np.testing.assert_array_equal(host(a.fat.counters), host(b.fat.counters))
    np.testing.assert_array_equal(host(a.slim.increment_counts), host(b.slim.increment_counts))


@pytest.mark.parametrize("variant", ("sff", "sf1", "sf2", "cm", "cu"))
def test_concurrent_sketches_on_two_streams_and_threads(variant):
    """The C ABI keeps no state between calls (include/sfsketch_cuda.h): two
    sketches updated at the same time from two host threads on two streams
    end in the same state as when updated one after the other."""
    import threading

    def streams(seed):
        c = W.cfg2(seed=seed, n=300_000, v=20_000)
        return [(c["ops"][a:a + 100_000], c["keys"][a:a + 100_000]) for a in (0, 100_000, 200_000)]

    def run(sk, batches, errs):
        try:
            with torch.cuda.stream(torch.cuda.Stream()):
                for ops, keys in batches:
                    sk.apply_ops(ops, keys)
                torch.cuda.current_stream().synchronize()
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    data = [streams(11), streams(12)]
    serial = [make_sketch(variant, 4, 4096, 4, 16384, 3 + i) for i in range(2)]
    for sk, b in zip(serial, data):
        run(sk, b, [])
    conc = [make_sketch(variant, 4, 4096, 4, 16384, 3 + i) for i in range(2)]
    errs = []
    th = [threading.Thread(target=run, args=(sk, b, errs)) for sk, b in zip(conc, data)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize()
    assert not errs, errs
    for a, b in zip(serial, conc):
        np.testing.assert_array_equal(host(a.counters if variant in ("cm", "cu") else a.slim.counters),
                                      host(b.counters if variant in ("cm", "cu") else b.slim.counters))


@pytest.mark.parametrize("variant", ("sff", "sf4"))
def test_sf_apply_replays_from_a_cuda_graph(variant):
    """A single-chunk SF apply does not synchronise the host or allocate
    (INTEGRATION.md §2), so it can be captured once in a CUDA graph and
    replayed: each replay applies the batch again, bit-exact with direct
    applies."""
    from paper_1701_04148_b200._ops import normalize_stream

    c = W.cfg2(seed=21, n=200_000, v=30_000)
    ops = np.concatenate([c["ops"], np.ones(40_000, dtype=np.uint8)])
    keys = np.concatenate([c["keys"], c["keys"][:40_000]])
    ops_d, keys_d = torch.as_tensor(ops).cuda(), torch.as_tensor(keys).cuda()
    ref = make_sketch(variant, 4, 4096, 4, None, 9)
    sk = make_sketch(variant, 4, 4096, 4, None, 9)
    ops_t, kb = normalize_stream(ops_d, keys_d)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        sk._submit(ops_t, kb)  # first application, and the workspace is allocated outside the capture
    torch.cuda.synchronize()
    ref.apply_ops(ops_d, keys_d)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        res = sk._submit(ops_t, kb)
    for _ in range(2):
        g.replay()
        torch.cuda.synchronize()
        ref.apply_ops(ops_d, keys_d)
        assert res.cpu().tolist()[0] == 0
        np.testing.assert_array_equal(host(sk.slim.counters), host(ref.slim.counters))
        np.testing.assert_array_equal(host(sk.fat.counters), host(ref.fat.counters))
        np.testing.assert_array_equal(host(sk.slim.increment_counts), host(ref.slim.increment_counts))


@pytest.mark.parametrize("kind", ("sff", "sf4", "sf3", "sf2", "sf1", "cm", "cu"))
def test_tiny_batches_both_engines_match_oracle(oracle, kind):
    """Batches of 1..40 ops, with the small-batch threshold at its default
    (<= 32 ops: the one-launch one-thread engine) and off (always the parallel
    pipeline): both end every batch in the oracle's state, including a
    phantom delete that aborts a batch part way."""
    from paper_1701_04148_b200 import _lib

    L = _lib.lib()
    assert L.sfk_small_batch_ops(-1) == 32
    c = W.cfg3(seed=77, n_ins=900, v=60, alpha=1.2)
    ops, keys = c["ops"].copy(), c["keys"].copy()
    if kind in ("sf1", "cu", "cm"):
        ops[:] = 0
    else:
        ops[500], keys[500] = 1, 0xFFFFFFFF  # a phantom: never inserted
    wp = {"sf3": 4 * 16, "sf1": 64, "sf2": 64}.get(kind)
    sizes = [1, 2, 3, 5, 8, 13, 21, 31, 32, 33, 40] * 6
    # (one-thread, warp-engine, block-engine thresholds): the one-thread
    # engine, the warp engine and the block engine (SFF / SF4 only), the
    # parallel pipeline
    for small, warp, block in ((32, 0, 0), (0, 2048, 0), (0, 0, 2048), (0, 0, 0)):
        prev = L.sfk_small_batch_ops(small)
        prev_w = L.sfk_warp_batch_ops(warp)
        prev_b = L.sfk_block_batch_ops(block)
        try:
            o = oracle.OracleSketch(kind, 3, 16, 4, wp, 5)
            sk = make_sketch(kind, 3, 16, 4, wp, 5)
            a = 0
            for n in sizes:
                b = min(a + n, len(ops))
                if a >= b:
                    break
                st = o.apply_ops(ops[a:b], keys[a:b].astype(np.uint64))
                assert apply_batches(sk, ops[a:b], keys[a:b]) == st[:2], (small, warp, block, a, b)
                assert_state_equal(sk, o.slim, o.inc, o.seen, o.fat if kind not in ("cm", "cu") else None)
                a = b
        finally:
            L.sfk_small_batch_ops(prev)
            L.sfk_warp_batch_ops(prev_w)
            L.sfk_block_batch_ops(prev_b)


def _state(sk):
    if isinstance(sk, P.SfSketch):
        parts = [sk.slim.counters, sk.slim.increment_counts, sk.fat.counters]
        if sk.deletion_sub is not None:
            parts.append(sk.deletion_sub.counters)
        return [host(p).copy() for p in parts] + [sk.slim.insertions_seen]
    return [host(sk.counters).copy(), host(sk.increment_counts).copy(), sk.insertions_seen]


@pytest.mark.parametrize("kind", ALL + ("cm", "cu"))
@pytest.mark.parametrize("n,bad_at", [(5, 3), (40, 0), (5000, 4321), (5000, 1)])
@pytest.mark.parametrize("sequential", [False, True])
@pytest.mark.parametrize("code", [2, 255])
def test_bad_op_codes_reject_the_whole_batch_on_the_device(kind, n, bad_at, sequential, code):
    """An op code other than 0 / 1 anywhere in the batch: ConfigurationError
    with the reference's message (_ops.py:27-34) and nothing applied, ops
    before it included. The SF / CM / CU applies check the codes on the device
    (status SFK_BAD_OPCODE) on the one-thread engine (<= 32 ops or
    sequential=True) and on the parallel pipeline alike."""
    from paper_1701_04148_b200.errors import ConfigurationError

    sk = make_sketch(kind, 4, 256, 4, 1024, 11)
    rng = np.random.default_rng(n + bad_at)
    warm = rng.integers(0, 1000, size=3000, dtype=np.uint64)
    sk.apply_ops(np.zeros(warm.size, np.uint8), warm)
    before = _state(sk)
    keys = torch.from_numpy(rng.choice(warm, size=n)).cuda()
    ops = torch.zeros(n, dtype=torch.uint8, device="cuda")
    ops[bad_at] = code
    with pytest.raises(ConfigurationError, match="op codes must be 0"):
        sk.apply_ops(ops, keys, sequential=sequential)
    for a, b in zip(before, _state(sk)):
        np.testing.assert_array_equal(a, b)
    # the sketch is still usable, and a fresh sketch that only saw a rejected
    # batch may still switch to the oracle-assisted mode
    ops[bad_at] = 0
    sk.apply_ops(ops, keys, sequential=sequential)
    if isinstance(sk, P.SfSketch):
        fresh = make_sketch(kind, 4, 256, 4, 1024, 11)
        bad = torch.full((3,), 7, dtype=torch.uint8, device="cuda")
        with pytest.raises(ConfigurationError):
            fresh.apply_ops(bad, torch.arange(3, dtype=torch.int64, device="cuda"))
        fresh.oracle_assisted_insert(5, 1)
        assert fresh.query(5) == 1


@pytest.mark.parametrize("seed", range(24))
def test_warp_engine_matches_oracle(oracle, seed):
    """The warp-cooperative small-batch engine (SFF / SF4, d x z <= 32 after
    rounding z up to a power of two) against the oracle: random shapes,
    Zipf-skewed keys (repeated buckets back to back), deletes including
    phantoms, fat presets near 2^32 (saturation), u32 / u64 / record keys,
    several batches; states equal after every batch."""
    from paper_1701_04148_b200 import _lib

    L = _lib.lib()
    rng = np.random.default_rng(9100 + seed)
    kind = ("sff", "sf4")[seed % 2]
    d = int(rng.integers(1, 9))
    z = int(rng.integers(1, 9))
    while d * (1 << (z - 1).bit_length()) > 32:
        z = max(1, z // 2)
    w = int(rng.choice([7, 64, 1000, 65536]))
    n = int(rng.integers(1, 3000))
    vocab = rng.integers(0, 1 << 62, size=int(rng.integers(1, 200)), dtype=np.uint64)
    ranks = np.minimum(rng.zipf(1.3, size=n) - 1, vocab.size - 1)
    keys = vocab[ranks]
    ops = np.zeros(n, np.uint8)
    dm = rng.random(n) < rng.choice([0.0, 0.2, 0.45])
    ops[dm] = 1
    o = oracle.OracleSketch(kind, d, w, z, None, seed)
    sk = make_sketch(kind, d, w, z, None, seed)
    if seed % 3 == 0:  # near saturation
        o.fat[...] = np.uint32(0xFFFFFFFF - 50)
        sk.fat.counters.fill_(0xFFFFFFFF - 50)
    kk = rng.integers(0, 3)
    if kk == 1:
        keys_in = (keys & np.uint64(0xFFFFFFFF)).astype(np.uint32)
        keys_o = keys_in.astype(np.uint64)
    elif kk == 2:
        recs = rng.integers(0, 256, size=(vocab.size, 13), dtype=np.uint8)[ranks]
        keys_in, keys_o = recs, oracle.keys_from_records(recs)
    else:
        keys_in, keys_o = keys, keys
    prev = L.sfk_warp_batch_ops(1 << 20)
    try:
        bounds = np.unique(np.concatenate([[0, n], rng.integers(0, n, size=3)]))
        for a, b in zip(bounds[:-1], bounds[1:]):
            st = o.apply_ops(ops[a:b], keys_o[a:b])
            got = apply_batches(sk, ops[a:b], keys_in[a:b])
            assert got == st[:2], (a, b)
            assert_state_equal(sk, o.slim, o.inc, o.seen, o.fat)
            if st[0] != 0:
                break
    finally:
        L.sfk_warp_batch_ops(prev)


@pytest.mark.parametrize("seed", range(32))
def test_block_engine_matches_oracle(oracle, seed):
    """The one-CTA block engine (SFF / SF4 batches of up to 8192 (op, row)
    pairs, z <= 8) against the oracle: random shapes (d 1-8, z 1-8, odd
    widths), Zipf-skewed keys (long same-cell chains in the dataflow
    replay), deletes including phantoms, fat presets near 2^32 (saturation),
    u32 / u64 / record keys, batch splits; one launch per batch and states
    equal after every batch."""
    from paper_1701_04148_b200 import _lib

    L = _lib.lib()
    rng = np.random.default_rng(9300 + seed)
    kind = ("sff", "sf4")[seed % 2]
    d = int(rng.choice([1, 2, 3, 4, 4, 4, 5, 8]))
    z = int(rng.choice([1, 2, 3, 4, 4, 5, 7, 8]))
    w = int(rng.choice([5, 64, 1000, 12800, 65536]))
    nmax = 8192 // d
    n = int(rng.integers(nmax // 4, nmax + 1))
    vocab = rng.integers(0, 1 << 62, size=int(rng.integers(1, 400)), dtype=np.uint64)
    ranks = np.minimum(rng.zipf(rng.choice([1.1, 1.3, 2.0]), size=n) - 1, vocab.size - 1)
    keys = vocab[ranks]
    ops = np.zeros(n, np.uint8)
    ops[rng.random(n) < rng.choice([0.0, 0.2, 0.45])] = 1
    o = oracle.OracleSketch(kind, d, w, z, None, seed)
    sk = make_sketch(kind, d, w, z, None, seed)
    if seed % 4 == 1:  # near saturation
        o.fat[...] = np.uint32(0xFFFFFFFF - 40)
        sk.fat.counters.fill_(0xFFFFFFFF - 40)
    kk = seed % 3
    if kk == 1:
        keys_in = (keys & np.uint64(0xFFFFFFFF)).astype(np.uint32)
        keys_o = keys_in.astype(np.uint64)
    elif kk == 2:
        recs = rng.integers(0, 256, size=(vocab.size, 13), dtype=np.uint8)[ranks]
        keys_in, keys_o = recs, oracle.keys_from_records(recs)
    else:
        keys_in, keys_o = keys, keys
    prev_w, prev_b = L.sfk_warp_batch_ops(0), L.sfk_block_batch_ops(1 << 20)
    try:
        bounds = np.unique(np.concatenate([[0, n], rng.integers(0, n, size=2)]))
        for a, b in zip(bounds[:-1], bounds[1:]):
            st = o.apply_ops(ops[a:b], keys_o[a:b])
            l0 = L.sfk_launch_count()
            got = apply_batches(sk, ops[a:b], keys_in[a:b])
            assert L.sfk_launch_count() - l0 == 1  # the block engine, one launch
            assert got == st[:2], (a, b)
            assert_state_equal(sk, o.slim, o.inc, o.seen, o.fat)
            if st[0] != 0:
                break
    finally:
        L.sfk_warp_batch_ops(prev_w)
        L.sfk_block_batch_ops(prev_b)


def test_block_engine_bad_opcode_and_limits(oracle):
    """A bad op code rejects the batch before anything is applied; batches past
    8192 (op, row) pairs or z > 8 take another engine (same results)."""
    from paper_1701_04148_b200 import _lib
    from paper_1701_04148_b200.errors import ConfigurationError

    L = _lib.lib()
    prev_w, prev_b = L.sfk_warp_batch_ops(0), L.sfk_block_batch_ops(1 << 20)
    try:
        sk = make_sketch("sff", 4, 1024, 4, None, 1)
        ops = np.zeros(1000, np.uint8)
        ops[700] = 3
        with pytest.raises(ConfigurationError):
            sk.apply_ops(ops, np.arange(1000, dtype=np.uint64))
        assert int(sk.fat.counters.sum()) == 0 and int(sk.slim.counters.sum()) == 0
        for d, z, n in ((4, 4, 2049), (2, 12, 500), (2, 33, 500), (8, 2, 1025)):
            rng = np.random.default_rng(d * z)
            keys = rng.integers(0, 300, size=n).astype(np.uint64)
            ops = (rng.random(n) < 0.1).astype(np.uint8)
            ops[: n // 2] = 0
            o = oracle.OracleSketch("sff", d, 4096, z, None, 2)
            sk = make_sketch("sff", d, 4096, z, None, 2)
            st = o.apply_ops(ops, keys)
            l0 = L.sfk_launch_count()
            assert apply_batches(sk, ops, keys) == st[:2]
            if z <= 8:  # (z > 8 runs on the one-thread engine: one launch too)
                assert L.sfk_launch_count() - l0 > 1  # not the block engine
            assert_state_equal(sk, o.slim, o.inc, o.seen, o.fat)
    finally:
        L.sfk_warp_batch_ops(prev_w)
        L.sfk_block_batch_ops(prev_b)


@pytest.mark.parametrize("case", ["u64", "i64_neg", "u32", "i32_neg", "u16", "bool", "pylist_big", "records", "tensor_cpu"])
def test_pinned_staging_matches_device_path(oracle, case):
    """Small HOST batches are staged in pinned memory and read in place by
    the kernels; every key dtype the reference accepts must give the same
    state as the device-tensor path (normalize_keys' cast rules) and the
    oracle."""
    rng = np.random.default_rng(len(case))
    n = 300
    ops = np.zeros(n, np.uint8)
    if case == "u64":
        keys = rng.integers(0, 1 << 63, size=n, dtype=np.uint64) * np.uint64(2)
    elif case == "i64_neg":
        keys = rng.integers(-(1 << 62), 1 << 62, size=n, dtype=np.int64)
    elif case == "u32":
        keys = rng.integers(0, 1 << 32, size=n, dtype=np.uint64).astype(np.uint32)
    elif case == "i32_neg":
        keys = rng.integers(-(1 << 31), 1 << 31, size=n, dtype=np.int64).astype(np.int32)
    elif case == "u16":
        keys = rng.integers(0, 1 << 16, size=n).astype(np.uint16)
    elif case == "bool":
        keys = rng.random(n) < 0.5
    elif case == "pylist_big":
        keys = [int(x) for x in rng.integers(1 << 62, (1 << 63) - 1, size=n, dtype=np.int64) * 2 + 1]
    elif case == "records":
        keys = rng.integers(0, 256, size=(n, 13), dtype=np.uint8)
    else:
        keys = torch.from_numpy(rng.integers(0, 1 << 40, size=n, dtype=np.int64))
    staged = make_sketch("sff", 4, 4096, 4, None, 3)
    staged.apply_ops(ops, keys)  # host input: pinned staging
    dev = make_sketch("sff", 4, 4096, 4, None, 3)
    from paper_1701_04148_b200._ops import normalize_keys

    kb = normalize_keys(keys)  # the device path's cast
    dev.apply_ops(torch.from_numpy(ops).cuda(), kb)
    np.testing.assert_array_equal(host(staged.slim.counters), host(dev.slim.counters))
    np.testing.assert_array_equal(host(staged.fat.counters), host(dev.fat.counters))
    if case == "records":
        ko = oracle.keys_from_records(keys)
    else:
        ko = np.asarray(kb.tensor.cpu().numpy()).astype(np.uint64)
    o = oracle.OracleSketch("sff", 4, 4096, 4, None, 3)
    o.apply_ops(ops, ko)
    np.testing.assert_array_equal(host(staged.slim.counters), o.slim)
    # a phantom delete on a staged batch raises with the reference's message and key
    with pytest.raises(P.PhantomDeletionError):
        staged.apply_ops(np.ones(1, np.uint8), np.array([12345678901], np.uint64))
