"""Host-buffer queries (sfk_min_query_host, SfSketch.query_many_host): host
keys in, host int64 estimates out, as the reference's query_many
(_kernels.py:229-241, sf.py:189-193). Every wire format (int64, u32, u16
codes over the slim's distinct large values), the automatic choice and its
u32 fallback, pinned and pageable buffers, chunk tails and ring wrap-around,
all three key kinds and the direct-int64 chunks, each against the oracle's
min_query (the restatement of _kernels.min_query)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_1701_04148_b200 as P  # noqa: E402
from paper_1701_04148_b200 import _lib  # noqa: E402
from paper_1701_04148_b200.errors import ConfigurationError  # noqa: E402
from paper_1701_04148_b200.hashing import seed_array  # noqa: E402
from paper_1701_04148_b200.sf import query_min_host  # noqa: E402

U32MAX = 0xFFFFFFFF


@pytest.fixture
def hq():
    """Restore the host-query knobs after each test."""
    L = _lib.lib()
    keys = (_lib.HQ_CHUNK, _lib.HQ_WIRE, _lib.HQ_DIRECT, _lib.HQ_RING)
    prev = {k: L.sfk_host_query_config(k, -1) for k in keys}
    yield L
    for k, v in prev.items():
        L.sfk_host_query_config(k, v)


def slim_with_large(rng, d, w, n_large_distinct, hot_frac=0.3):
    """Counters mostly small, a fraction of cells drawn from n_large_distinct
    values >= 0xF800 (including U32MAX)."""
    c = rng.integers(0, 5000, size=(d, w), dtype=np.int64).astype(np.uint32)
    if n_large_distinct:
        large = np.unique(rng.integers(0xF800, U32MAX, size=4 * n_large_distinct, dtype=np.int64))
        large = rng.permutation(large)[: n_large_distinct - 1].astype(np.uint32)
        large = np.concatenate([large, np.array([U32MAX], np.uint32)])
        assert np.unique(large).size == n_large_distinct
        m = rng.random((d, w)) < hot_frac
        m.flat[: n_large_distinct] = True  # every large value is present
        picks = large[rng.integers(0, large.size, size=int(m.sum()))]
        picks[: n_large_distinct] = large
        c[m] = picks
    return c


def keys_for(rng, kind, n):
    if kind == "u32":
        return rng.integers(0, 1 << 32, size=n, dtype=np.uint64).astype(np.uint32)
    if kind == "u64":
        return rng.integers(0, 1 << 63, size=n, dtype=np.uint64) * np.uint64(2) + np.uint64(1)
    return rng.integers(0, 256, size=(n, 13), dtype=np.uint8)


def oracle_keys(orc, kind, keys):
    return orc.keys_from_records(keys) if kind == "rec" else keys.astype(np.uint64)


@pytest.mark.parametrize("wire", [_lib.WIRE_AUTO, _lib.WIRE_I64, _lib.WIRE_U32, _lib.WIRE_C16])
@pytest.mark.parametrize("kind", ["u32", "u64", "rec"])
@pytest.mark.parametrize("pinned", [False, True])
def test_host_query_wires(oracle, hq, wire, kind, pinned):
    rng = np.random.default_rng(7 + wire * 10 + len(kind) + pinned)
    d, w = 4, 65536
    c = slim_with_large(rng, d, w, 300)
    seeds = seed_array(11, 0, d)
    n = 3 * 65536 + 4097  # several chunks, a ragged tail, ring wrap-around
    keys = keys_for(rng, kind, n)
    hq.sfk_host_query_config(_lib.HQ_CHUNK, 65536)
    hq.sfk_host_query_config(_lib.HQ_RING, 2)
    hq.sfk_host_query_config(_lib.HQ_WIRE, wire)
    kt = torch.from_numpy(keys)
    out = torch.full((n,), -5, dtype=torch.int64)
    if pinned:
        kt, out = kt.pin_memory(), out.pin_memory()
    counters = torch.from_numpy(c).cuda()
    query_min_host(counters, seeds, kt, out)
    want = oracle.min_query(c, seeds, oracle_keys(oracle, kind, keys), threads=oracle.max_threads())
    np.testing.assert_array_equal(out.numpy(), want)
    used = hq.sfk_host_query_config(_lib.HQ_LAST_WIRE, -1)
    assert used == (_lib.WIRE_C16 if wire == _lib.WIRE_AUTO else wire)


@pytest.mark.parametrize("n_large,expect", [(0, _lib.WIRE_C16), (2048, _lib.WIRE_C16), (2049, _lib.WIRE_U32)])
def test_host_query_dictionary_limit(oracle, hq, n_large, expect):
    """code16 holds at most 2048 distinct values >= 0xF800; one more falls back to u32."""
    rng = np.random.default_rng(n_large)
    d, w = 4, 32768
    c = slim_with_large(rng, d, w, n_large, hot_frac=0.5)
    seeds = seed_array(5, 0, d)
    keys = keys_for(rng, "u32", 500_000)
    hq.sfk_host_query_config(_lib.HQ_CHUNK, 1 << 17)
    out = query_min_host(torch.from_numpy(c).cuda(), seeds, keys)
    np.testing.assert_array_equal(out.numpy(), oracle.min_query(c, seeds, keys.astype(np.uint64),
                                                                threads=oracle.max_threads()))
    assert hq.sfk_host_query_config(_lib.HQ_LAST_WIRE, -1) == expect
    if n_large:
        assert int(out.max()) >= 0xF800  # the large codes were exercised


@pytest.mark.parametrize("direct", [1, 2, 3])
def test_host_query_direct_chunks(oracle, hq, direct):
    """Every direct-th chunk returns int64 over the link into a pinned output."""
    rng = np.random.default_rng(direct)
    d, w = 4, 65536
    c = slim_with_large(rng, d, w, 40)
    seeds = seed_array(3, 0, d)
    n = 5 * 65536 + 17
    keys = torch.from_numpy(keys_for(rng, "u32", n)).pin_memory()
    out = torch.empty(n, dtype=torch.int64).pin_memory()
    hq.sfk_host_query_config(_lib.HQ_CHUNK, 65536)
    hq.sfk_host_query_config(_lib.HQ_DIRECT, direct)
    query_min_host(torch.from_numpy(c).cuda(), seeds, keys, out)
    np.testing.assert_array_equal(out.numpy(), oracle.min_query(c, seeds, keys.numpy().astype(np.uint64),
                                                                threads=oracle.max_threads()))


@pytest.mark.parametrize("d,w", [(1, 1000), (3, 12800), (4, 65536), (8, 4096), (5, 1 << 16)])
@pytest.mark.parametrize("n", [1, 7, 4096, 100_003])
def test_host_query_shapes(oracle, hq, d, w, n):
    rng = np.random.default_rng(d * 1000 + n)
    c = slim_with_large(rng, d, w, 16, hot_frac=0.05)
    seeds = seed_array(9, 0, d)
    keys = keys_for(rng, "u64", n)
    out = query_min_host(torch.from_numpy(c).cuda(), seeds, keys)
    np.testing.assert_array_equal(out.numpy(), oracle.min_query(c, seeds, keys, threads=oracle.max_threads()))


def test_query_many_host_matches_device(hq):
    """SfSketch.query_many_host on a built cfg-3-shaped slim equals query_many."""
    from paper_1701_04148_b200 import workloads as W

    c = W.cfg3(seed=2017, n_ins=400_000, v=50_000, alpha=1.0)
    sk = P.SfSketch(P.SketchParams(d=4, w=65536, z=4, master_seed=2017), "sff")
    sk.apply_ops(c["ops"], c["keys"])
    q = np.concatenate([c["distinct"], np.arange(1, 300_001, dtype=np.uint32) * np.uint32(2654435761)])
    res = sk.query_many_host(q)
    assert isinstance(res, np.ndarray) and res.dtype == np.int64
    np.testing.assert_array_equal(res, sk.query_many(q).cpu().numpy())
    out = torch.empty(q.size, dtype=torch.int64)
    assert sk.query_many_host(torch.from_numpy(q), out=out) is out
    np.testing.assert_array_equal(out.numpy(), res)
    cm = P.CmSketch(P.SketchParams(d=4, w=65536, master_seed=3))
    cm.apply_ops(c["ops"][c["ops"] == 0], c["keys"][c["ops"] == 0])
    np.testing.assert_array_equal(cm.query_many_host(q), cm.query_many(q).cpu().numpy())


def test_host_query_empty_and_errors(hq):
    sk = P.SfSketch(P.SketchParams(d=4, w=1024, z=4, master_seed=1), "sff")
    assert sk.query_many_host(np.zeros(0, np.uint32)).shape == (0,)
    with pytest.raises(ConfigurationError):
        sk.query_many_host(np.zeros(4, np.uint32), out=torch.empty(3, dtype=torch.int64))
    with pytest.raises(ConfigurationError):
        sk.query_many_host(torch.zeros(4, dtype=torch.uint32, device="cuda"))
    with pytest.raises(ConfigurationError):
        sk.query_many_host(np.zeros((2, 2), np.uint32))


@pytest.mark.parametrize("kind", ["u32", "u64", "rec"])
@pytest.mark.parametrize("staged_n", [0, 1, 65536, 2 * 65536 + 5, 3 * 65536 + 4097])
@pytest.mark.parametrize("pinned", [False, True])
def test_host_query_staged_prefix(oracle, hq, kind, staged_n, pinned):
    """stage_query_keys + query_min_host(staged=...): chunks wholly inside the
    device-resident prefix are queried in place, the partly staged chunk and
    the rest through the H2D ring; same estimates as the unstaged path."""
    rng = np.random.default_rng(staged_n + len(kind) + 100 * pinned)
    d, w = 4, 65536
    c = slim_with_large(rng, d, w, 300)
    seeds = seed_array(11, 0, d)
    n = 3 * 65536 + 4097
    keys = keys_for(rng, kind, n)
    hq.sfk_host_query_config(_lib.HQ_CHUNK, 65536)
    hq.sfk_host_query_config(_lib.HQ_RING, 2)
    kt = torch.from_numpy(keys)
    out = torch.full((n,), -5, dtype=torch.int64)
    if pinned:
        kt, out = kt.pin_memory(), out.pin_memory()
    counters = torch.from_numpy(c).cuda()
    st = P.sf.stage_query_keys(kt, staged_n)
    assert st.n == staged_n
    query_min_host(counters, seeds, kt, out, staged=st)
    want = oracle.min_query(c, seeds, oracle_keys(oracle, kind, keys), threads=oracle.max_threads())
    np.testing.assert_array_equal(out.numpy(), want)


def test_host_query_staged_mismatch(hq):
    rng = np.random.default_rng(1)
    c = torch.from_numpy(slim_with_large(rng, 4, 4096, 0)).cuda()
    seeds = seed_array(1, 0, 4)
    k32 = keys_for(rng, "u32", 1000)
    st = P.sf.stage_query_keys(k32)
    with pytest.raises(ConfigurationError):
        query_min_host(c, seeds, keys_for(rng, "u64", 1000), staged=st)  # other key type
    with pytest.raises(ConfigurationError):
        query_min_host(c, seeds, k32[:500], staged=st)  # prefix longer than the batch


def test_query_many_host_staged_during_build(hq):
    """The bench's e2e order: stage the query keys, build, then query."""
    from paper_1701_04148_b200 import workloads as W

    c = W.cfg3(seed=2017, n_ins=400_000, v=50_000, alpha=1.0)
    q = np.random.default_rng(3).integers(0, 1 << 32, size=1_000_000, dtype=np.uint64).astype(np.uint32)
    qh = torch.from_numpy(q).pin_memory()
    hq.sfk_host_query_config(_lib.HQ_CHUNK, 1 << 16)
    sk = P.SfSketch(P.SketchParams(d=4, w=65536, z=4, master_seed=2017), "sff")
    st = sk.stage_query_keys(qh, 600_000)
    sk.apply_ops(c["ops"], c["keys"])
    got = sk.query_many_host(qh, staged=st)
    want = sk.query_many(torch.from_numpy(q).cuda()).cpu()
    assert torch.equal(got, want)


def test_query_many_host_staged_with_next_apply(hq):
    """with_next_apply: the copy starts inside apply_ops, behind the batch's upload."""
    from paper_1701_04148_b200 import workloads as W

    c = W.cfg3(seed=2018, n_ins=300_000, v=40_000, alpha=1.2)
    q = np.random.default_rng(4).integers(0, 1 << 32, size=700_001, dtype=np.uint64).astype(np.uint32)
    qh = torch.from_numpy(q).pin_memory()
    hq.sfk_host_query_config(_lib.HQ_CHUNK, 1 << 16)
    sk = P.SfSketch(P.SketchParams(d=4, w=65536, z=4, master_seed=2018), "sff")
    st = sk.stage_query_keys(qh, 500_000, with_next_apply=True)
    assert st.event is None  # not yet issued
    sk.apply_ops(torch.from_numpy(c["ops"]).pin_memory(), torch.from_numpy(c["keys"]).pin_memory())
    assert st.event is not None
    got = sk.query_many_host(qh, staged=st)
    assert torch.equal(got, sk.query_many(torch.from_numpy(q).cuda()).cpu())
    # a deferred handle that no apply issued is issued by the query itself
    st2 = sk.stage_query_keys(qh, 300_000, with_next_apply=True)
    assert torch.equal(sk.query_many_host(qh, staged=st2), got)
