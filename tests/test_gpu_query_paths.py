"""Every point-query kernel path (L2 gathers, whole table in shared memory,
row-partitioned cluster with DSMEM min-reduction, and its warp-pipelined
form with TMA key rings) against the oracle's
min_query (the restatement of _kernels.min_query, _kernels.py:229-241), with
the path forced through sfk_query_path. Covers the cluster path's u16 rows
with the exact >= 65535 re-gather, u32 rows, odd d, non-power-of-two widths,
tile tails, misaligned key / output pointers and all three key kinds."""

import ctypes

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_1701_04148_b200 import _lib  # noqa: E402
from paper_1701_04148_b200.hashing import seed_array  # noqa: E402

L2, SMEM, CLUSTER, CW = 1, 2, 3, 4


def run_query(counters, seeds, keys_t, kind, rec, n, out_t, path):
    L = _lib.lib()
    prev = L.sfk_query_path(path)
    try:
        rc = L.sfk_min_query(counters.data_ptr(), seeds.ctypes.data_as(ctypes.c_void_p), counters.shape[0],
                             counters.shape[1], keys_t.data_ptr(), kind, rec, n, out_t.data_ptr(),
                             _lib.stream_ptr())
        _lib.check(rc, "sfk_min_query")
        torch.cuda.synchronize()
        return L.sfk_query_last_path()
    finally:
        L.sfk_query_path(prev)


def table(rng, d, w, hi):
    c = rng.integers(0, hi, size=(d, w), dtype=np.uint64).astype(np.uint32)
    return c


@pytest.mark.parametrize("d,w,hi,path", [
    (4, 65536, 1 << 20, CLUSTER),   # cfg 3/5 shape: u16 rows, many clamped cells
    (4, 65536, 70000, CLUSTER),     # values straddling 65535
    (4, 65536, 1000, CLUSTER),      # no clamping at all
    (4, 16384, 1 << 32, CLUSTER),   # cfg 1 shape: u32 rows
    (3, 65536, 1 << 18, CLUSTER),   # odd cluster size
    (5, 12345, 1 << 32, CLUSTER),   # non-pow2 width, u32 rows
    (8, 50000, 1 << 17, CLUSTER),   # portable maximum cluster, u16 rows, non-pow2
    (2, 40000, 1 << 32, CLUSTER),
    (4, 12800, 1 << 32, SMEM),      # cfg 4 shape
    (4, 65536, 1 << 32, L2),
    (4, 65536, 1 << 20, CW),        # cfg 3/5 shape on the warp-pipelined kernel: u16 rows
    (4, 65536, 70000, CW),
    (4, 65536, 1000, CW),
    (4, 16384, 1 << 32, CW),        # u32 rows
    (8, 50000, 1 << 17, CW),        # d = 8 cluster, non-pow2 u16 rows
    (8, 8192, 1 << 32, CW),         # d = 8, u32 rows
    (2, 40000, 1 << 32, CW),        # d = 2, non-pow2, u32 rows
    (2, 65536, 1 << 18, CW),        # d = 2, u16 rows
])
@pytest.mark.parametrize("n", [1, 4097, 100_003, 1_000_000])
def test_query_paths_u32_keys(oracle, d, w, hi, path, n):
    rng = np.random.default_rng(d * 1000 + w + n)
    c = table(rng, d, w, hi)
    # make some cells exactly 65534 / 65535 / 65536 so every clamp edge is hit
    c.flat[rng.integers(0, c.size, 512)] = rng.choice(np.array([65534, 65535, 65536], np.uint32), 512)
    seeds = seed_array(7 + d, 0, d)
    keys = rng.integers(0, 1 << 32, size=n, dtype=np.uint64).astype(np.uint32)
    ct = torch.from_numpy(c).cuda()
    kt = torch.from_numpy(keys).cuda()
    out = torch.full((n,), -1, dtype=torch.int64, device="cuda")
    took = run_query(ct, seeds, kt, _lib.KEY_U32, 0, n, out, path)
    # the warp-pipelined kernel needs one whole warp-tile (>= 512 keys);
    # below that the request falls back to the CTA-level cluster kernel
    assert took == (CLUSTER if path == CW and n < 512 else path)
    want = oracle.min_query(c, seeds, keys.astype(np.uint64))
    np.testing.assert_array_equal(out.cpu().numpy(), want)


@pytest.mark.parametrize("path", [CLUSTER, CW])
@pytest.mark.parametrize("n_hot,distinct_vals", [(300, 0), (300, 7), (1000, 0), (3000, 0)])
def test_cluster_hot_keys_take_the_exact_regather(oracle, n_hot, distinct_vals, path):
    """Keys whose every row counter is large (the hot keys of a Zipf stream)
    must come back with their exact u32 minimum: through the cluster-wide
    rank codes (few large cells, ties across rows when distinct_vals > 0)
    or, when the overflow tables run out, through the per-row decode."""
    d, w = 4, 65536
    rng = np.random.default_rng(3 + n_hot + distinct_vals)
    seeds = seed_array(2017, 0, d)
    keys = rng.integers(0, 1 << 32, size=300_000, dtype=np.uint64).astype(np.uint32)
    c = rng.integers(0, 60000, size=(d, w), dtype=np.uint64).astype(np.uint32)
    hot = keys[:n_hot].astype(np.uint64)
    pool = 63488 + rng.integers(0, 1 << 20, size=max(distinct_vals, 1)).astype(np.uint32)
    for i in range(d):
        idx = oracle.min_query(np.arange(w, dtype=np.uint32)[None, :].repeat(1, 0), seeds[i:i + 1], hot)
        if distinct_vals:
            c[i, idx] = rng.choice(pool, size=idx.size)
        else:
            c[i, idx] = 63488 + rng.integers(0, 1 << 20, size=idx.size).astype(np.uint32)
    ct = torch.from_numpy(c).cuda()
    kt = torch.from_numpy(keys).cuda()
    out = torch.empty(keys.size, dtype=torch.int64, device="cuda")
    assert run_query(ct, seeds, kt, _lib.KEY_U32, 0, keys.size, out, path) == path
    got = out.cpu().numpy()
    want = oracle.min_query(c, seeds, keys.astype(np.uint64))
    np.testing.assert_array_equal(got, want)
    assert (got[:n_hot] >= 63488).all()


@pytest.mark.parametrize("path", [L2, CLUSTER, CW])
def test_query_paths_misaligned_views(oracle, path):
    d, w, n = 4, 65536, 200_001
    rng = np.random.default_rng(11)
    c = table(rng, d, w, 1 << 17)
    seeds = seed_array(1, 0, d)
    keys = rng.integers(0, 1 << 32, size=n + 3, dtype=np.uint64).astype(np.uint32)
    kt = torch.from_numpy(keys).cuda()[1:n + 1]          # 4-B aligned only
    out_base = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    out = out_base[1:]                                   # 8-B aligned only
    ct = torch.from_numpy(c).cuda()
    # misaligned views cannot feed the bulk copies: CW falls back to CLUSTER
    assert run_query(ct, seeds, kt, _lib.KEY_U32, 0, n, out, path) == (CLUSTER if path == CW else path)
    np.testing.assert_array_equal(out.cpu().numpy(), oracle.min_query(c, seeds, keys[1:n + 1].astype(np.uint64)))


@pytest.mark.parametrize("d,w,hi", [(4, 65536, 1 << 20), (4, 65536, 70000), (4, 16384, 1 << 32), (8, 50000, 1 << 17),
                                    (2, 65536, 1 << 18)])
@pytest.mark.parametrize("n", [1000, 100_003, 3_000_001])
def test_warp_pipelined_cluster_u64_keys(oracle, d, w, hi, n):
    """The reference's own key dtype (uint64) on the warp-pipelined kernel:
    full 64-bit keys hashed with the 64-bit form of the row reduction."""
    rng = np.random.default_rng(d * 7 + w + n)
    c = table(rng, d, w, hi)
    c.flat[rng.integers(0, c.size, 512)] = rng.choice(np.array([65534, 65535, 65536], np.uint32), 512)
    seeds = seed_array(17 + d, 0, d)
    k64 = rng.integers(0, np.iinfo(np.uint64).max, size=n, dtype=np.uint64)
    out = torch.full((n,), -1, dtype=torch.int64, device="cuda")
    took = run_query(torch.from_numpy(c).cuda(), seeds, torch.from_numpy(k64).cuda(), _lib.KEY_U64, 0, n, out, CW)
    assert took == CW
    np.testing.assert_array_equal(out.cpu().numpy(), oracle.min_query(c, seeds, k64))


@pytest.mark.parametrize("path", [L2, SMEM, CLUSTER])
def test_query_paths_u64_and_record_keys(oracle, path):
    d, w, n = 4, 16384 if path != SMEM else 12800, 150_000
    rng = np.random.default_rng(5)
    c = table(rng, d, w, 1 << 32)
    seeds = seed_array(99, 0, d)
    ct = torch.from_numpy(c).cuda()
    k64 = rng.integers(0, np.iinfo(np.uint64).max, size=n, dtype=np.uint64)
    out = torch.empty(n, dtype=torch.int64, device="cuda")
    assert run_query(ct, seeds, torch.from_numpy(k64).cuda(), _lib.KEY_U64, 0, n, out, path) == path
    np.testing.assert_array_equal(out.cpu().numpy(), oracle.min_query(c, seeds, k64))
    recs = rng.integers(0, 256, size=(n, 13), dtype=np.uint8)
    assert run_query(ct, seeds, torch.from_numpy(recs.reshape(-1)).cuda(), _lib.KEY_RECORD, 13, n, out,
                     path) == path
    np.testing.assert_array_equal(out.cpu().numpy(), oracle.min_query(c, seeds, oracle.keys_from_records(recs)))


def test_auto_path_picks_warp_pipelined_cluster_for_cfg5_shape():
    d, w, n = 4, 65536, 1 << 22
    c = torch.zeros((d, w), dtype=torch.uint32, device="cuda")
    seeds = seed_array(2017, 0, d)
    for dt, kind in ((torch.uint32, _lib.KEY_U32), (torch.uint64, _lib.KEY_U64)):
        keys = torch.zeros(n, dtype=dt, device="cuda")
        out = torch.empty(n, dtype=torch.int64, device="cuda")
        assert run_query(c, seeds, keys, kind, 0, n, out, 0) == CW
        assert int(out.max()) == 0


def two_phase(counters, seeds, keys_t, kind, n, out_t, stream=None, gather_stream=None):
    L = _lib.lib()
    d, w = counters.shape
    idx = torch.empty(d * max(n, 1), dtype=torch.uint16, device="cuda")
    s1 = _lib.stream_ptr(stream)
    _lib.check(L.sfk_query_index(seeds.ctypes.data_as(ctypes.c_void_p), d, w, keys_t.data_ptr(), kind, 0, n,
                                 idx.data_ptr(), s1), "sfk_query_index")
    if gather_stream is not None:
        gather_stream.wait_stream(stream)
    _lib.check(L.sfk_min_query_idx(counters.data_ptr(), d, w, idx.data_ptr(), n, out_t.data_ptr(),
                                   _lib.stream_ptr(gather_stream)), "sfk_min_query_idx")
    torch.cuda.synchronize()
    return L.sfk_query_last_path()


@pytest.mark.parametrize("d,w,hi", [(4, 65536, 1 << 17), (4, 65536, 70000), (3, 40000, 1 << 20), (2, 1024, 1 << 32),
                                    (5, 65536, 1000)])
@pytest.mark.parametrize("n", [1, 4097, 3_000_001, 4_194_304])
def test_two_phase_query_matches_oracle(oracle, d, w, hi, n):
    """sfk_query_index + sfk_min_query_idx == min_query (_kernels.py:229-241)."""
    rng = np.random.default_rng(d + w + n)
    c = table(rng, d, w, hi)
    seeds = seed_array(31 + d, 0, d)
    keys = rng.integers(0, 1 << 32, size=n, dtype=np.uint64).astype(np.uint32)
    out = torch.full((n,), -1, dtype=torch.int64, device="cuda")
    two_phase(torch.from_numpy(c).cuda(), seeds, torch.from_numpy(keys).cuda(), _lib.KEY_U32, n, out)
    np.testing.assert_array_equal(out.cpu().numpy(), oracle.min_query(c, seeds, keys.astype(np.uint64)))


def test_two_phase_index_overlaps_a_build(oracle):
    """The index pass reads no counters: it may run on another stream while
    the sketch is being built; the gathers after the build see the final slim."""
    import paper_1701_04148_b200 as P
    from paper_1701_04148_b200 import workloads as W

    c = W.cfg3(seed=4, n_ins=2_000_000, v=100_000, alpha=1.0)
    sk = P.SfSketch(P.SketchParams(d=4, w=65536, z=4, master_seed=4), "sff")
    q = W.query_keys(9, c["distinct"], 1.0, 0, 4_000_000)
    qt = torch.from_numpy(q).cuda()
    ops, keys = torch.from_numpy(c["ops"]).cuda(), torch.from_numpy(c["keys"]).cuda()
    torch.cuda.synchronize()
    side = torch.cuda.Stream()
    L = _lib.lib()
    idx = torch.empty(4 * q.size, dtype=torch.uint16, device="cuda")
    _lib.check(L.sfk_query_index(sk._slim_seeds.ctypes.data_as(ctypes.c_void_p), 4, 65536, qt.data_ptr(),
                                 _lib.KEY_U32, 0, q.size, idx.data_ptr(), _lib.stream_ptr(side)), "index")
    sk.apply_ops(ops, keys)  # current stream, concurrently
    torch.cuda.current_stream().wait_stream(side)
    out = torch.empty(q.size, dtype=torch.int64, device="cuda")
    _lib.check(L.sfk_min_query_idx(sk.slim.counters.data_ptr(), 4, 65536, idx.data_ptr(), q.size, out.data_ptr(),
                                   _lib.stream_ptr()), "gather")
    np.testing.assert_array_equal(out.cpu().numpy(), sk.query_many(qt).cpu().numpy())
    o = oracle.OracleSketch("sff", 4, 65536, 4, None, 4)
    o.apply_ops(c["ops"], c["keys"].astype(np.uint64))
    np.testing.assert_array_equal(out.cpu().numpy()[:200_000], o.query_many(q[:200_000].astype(np.uint64)))
