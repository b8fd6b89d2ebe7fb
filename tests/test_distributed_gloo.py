"""Multi-process (world_size 2, gloo, CPU) checks of the sharding logic:
contiguous shards, bit-exact uint32 count-min merge through int32 all-reduce
(with SaturationError on every rank when a merged counter would pass
2^32 - 1), slim broadcast, the global failure-free precheck, a sharded CM
build (oracle replicas per shard + merge) equal to one sequential build, and
distributed.sharded_cm_apply on a CPU stand-in sketch: a warm sketch with
cross-shard deletes, and a phantom delete that must raise the same error on
every rank. tests/test_gpu_distributed.py runs the same paths through the GPU
sketches."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1701_04148_b200 import distributed as PD
from paper_1701_04148_b200 import workloads as W


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def run2(fn):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, fn, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    return out


def _merge(rank, world):
    rng = np.random.Generator(np.random.PCG64(rank))
    c = torch.from_numpy(rng.integers(0, 1 << 31, size=(4, 64), dtype=np.uint64).astype(np.uint32))
    tallies = torch.tensor([rank + 1] * 4, dtype=torch.int64)
    mine = c.clone()
    seen = PD.allreduce_counters_(c, tallies, seen=10 * (rank + 1))
    return mine.numpy(), c.numpy(), tallies.numpy(), seen


def test_allreduce_sums_exactly():
    out = run2(_merge)
    want = out[0][0].astype(np.uint64) + out[1][0].astype(np.uint64)
    assert want.max() <= 0xFFFFFFFF
    for r in (0, 1):
        np.testing.assert_array_equal(out[r][1], want.astype(np.uint32))
        np.testing.assert_array_equal(out[r][2], [3, 3, 3, 3])
        assert out[r][3] == 30


def _merge_near_limit(rank, world):
    # both maxima near 2^32 - 1 but in different cells: the sum of maxima
    # exceeds the bound, the exact sums do not
    c = torch.zeros((2, 8), dtype=torch.uint32)
    c[0, rank] = 0xFFFFFFF0
    PD.allreduce_counters_(c, None, 0)
    return c.numpy()


def _merge_overflow(rank, world):
    c = torch.zeros((2, 8), dtype=torch.uint32)
    c[1, 3] = 0x80000000 + rank
    try:
        PD.allreduce_counters_(c, None, 0)
    except Exception as e:  # noqa: BLE001
        return type(e).__name__, str(e)
    return "no error", c.numpy()


def test_allreduce_checks_the_exact_sums_near_the_limit():
    out = run2(_merge_near_limit)
    for r in (0, 1):
        assert out[r][0, 0] == 0xFFFFFFF0 and out[r][0, 1] == 0xFFFFFFF0


def test_allreduce_overflow_raises_saturation_on_every_rank():
    out = run2(_merge_overflow)
    assert out[0][0] == out[1][0] == "SaturationError"
    assert out[0][1] == out[1][1]


def _bcast(rank, world):
    c = torch.full((4, 16), 7, dtype=torch.uint32) if rank == 0 else torch.zeros((4, 16), dtype=torch.uint32)
    c[0, 0] = 0xFFFFFFFF if rank == 0 else 0
    PD.broadcast_counters_(c, src=0)
    return c.numpy()


def test_broadcast_slim():
    out = run2(_bcast)
    np.testing.assert_array_equal(out[0], out[1])
    assert out[1][0, 0] == 0xFFFFFFFF


def _precheck(rank, world):
    ops = torch.zeros(1000, dtype=torch.uint8)
    ok_fresh = PD.batch_is_failure_free(torch.zeros((4, 8), dtype=torch.uint32), ops)
    near = torch.full((4, 8), 0xFFFFFFFF - 1500, dtype=torch.uint32)
    sat = PD.batch_is_failure_free(near, ops)  # 2 x 1000 inserts > 1500 headroom
    dels = torch.ones(10, dtype=torch.uint8)
    phantom = PD.batch_is_failure_free(torch.zeros((4, 8), dtype=torch.uint32), dels)
    return ok_fresh, sat, phantom


def test_global_precheck():
    out = run2(_precheck)
    for r in (0, 1):
        assert out[r] == (True, False, False)


def _sharded_cm(rank, world):
    from oracle import oracle as orc

    c = W.cfg2(seed=5, n=40_000, v=3_000)
    a, b = PD.shard_range(len(c["ops"]), rank, world)
    o = orc.OracleSketch("cm", 4, 1024, master_seed=5)
    o.apply_ops(c["ops"][a:b], c["keys"][a:b].astype(np.uint64))
    counters = torch.from_numpy(o.slim.copy())
    tallies = torch.from_numpy(o.inc.copy())
    seen = PD.allreduce_counters_(counters, tallies, o.seen)
    return counters.numpy(), tallies.numpy(), seen


def test_sharded_cm_build_equals_sequential(oracle):
    out = run2(_sharded_cm)
    c = W.cfg2(seed=5, n=40_000, v=3_000)
    full = oracle.OracleSketch("cm", 4, 1024, master_seed=5)
    full.apply_ops(c["ops"], c["keys"].astype(np.uint64))
    for r in (0, 1):
        np.testing.assert_array_equal(out[r][0], full.slim)
        np.testing.assert_array_equal(out[r][1], full.inc)
        assert out[r][2] == full.seen


@pytest.mark.parametrize("n,world", [(10, 3), (7, 7), (1_000_000_000, 8), (5, 8)])
def test_shard_range_partitions(n, world):
    spans = [PD.shard_range(n, r, world) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == n
    for (a0, b0), (a1, b1) in zip(spans, spans[1:]):
        assert b0 == a1 and a0 <= b0


class _CpuKeys:
    """KeyBatch stand-in for CPU tensors (u64 keys)."""

    def __init__(self, keys):
        self.tensor = keys
        self.n = int(keys.shape[0])
        self.kind, self.rec_len = 0, 0

    def slice(self, a, b):
        return _CpuKeys(self.tensor[a:b])

    def key_at(self, t):
        return int(self.tensor[t])


class _CpuCm:
    """Count-min replica on CPU tensors with the hooks sharded_cm_apply uses;
    the raw delta and the exact apply come from the oracle (test stand-ins for
    sfk_cm_delta / sfk_cm_apply)."""

    def __init__(self, d, w, seed):
        from oracle import oracle as orc
        from paper_1701_04148_b200.params import SketchParams

        self.orc = orc
        self.params = SketchParams(d=d, w=w, master_seed=seed)
        self._seeds = orc.seed_array(seed, 0, d)
        self.counters = torch.zeros((d, w), dtype=torch.uint32)
        self.increment_counts = torch.zeros(d, dtype=torch.int64)
        self.insertions_seen = 0

    def _normalize(self, ops, keys):
        return torch.as_tensor(np.asarray(ops, dtype=np.uint8)), _CpuKeys(np.asarray(keys, dtype=np.uint64))

    def _cm_delta_(self, delta, ops_t, kb):
        d, w = self.params.d, self.params.w
        sign = np.where(ops_t.numpy() == 0, 1, -1).astype(np.int64)
        acc = delta.numpy().view(np.int32).astype(np.int64)
        for i in range(d):
            j = self.orc.min_query(np.arange(w, dtype=np.uint32)[None, :], self._seeds[i:i + 1], kb.tensor)
            np.add.at(acc[i], j, sign)
        delta.copy_(torch.from_numpy((acc & 0xFFFFFFFF).astype(np.uint32)))

    def _submit(self, ops_t, kb):
        c = self.counters.numpy().copy()
        inc = self.increment_counts.numpy().copy()
        st = self.orc.cm_apply(c, self._seeds, ops_t.numpy(), kb.tensor, inc)
        self.counters.copy_(torch.from_numpy(c))
        self.increment_counts.copy_(torch.from_numpy(inc))
        return torch.tensor(list(st), dtype=torch.int64)

    @staticmethod
    def _raise_for_status(status, bad, kb):
        from paper_1701_04148_b200._ops import raise_for_status

        raise_for_status(status, bad, kb)


def _warm_stream(seed):
    """A warm-up batch and a main batch whose deletes (about 1/3 of its ops)
    target keys inserted in the warm-up or anywhere in the main batch, so
    under a 2-way split many deletes meet a key inserted in the other shard."""
    rng = np.random.default_rng(seed)
    keys = rng.integers(0, 1 << 40, size=300, dtype=np.uint64)
    warm = rng.choice(keys, size=3000)
    main_ins = rng.choice(keys, size=4000)
    # deletes of the warm keys, placed anywhere (never phantom: the warm-up
    # put every count high enough)
    dels = rng.choice(warm, size=2000)
    ops = np.concatenate([np.zeros(4000, np.uint8), np.ones(2000, np.uint8)])
    ks = np.concatenate([main_ins, dels])
    perm = rng.permutation(ops.size)
    return warm, ops[perm], ks[perm]


def _sharded_cm_fake(rank, world):
    warm, ops, keys = _warm_stream(11)
    sk = _CpuCm(4, 64, 3)
    st = sk._submit(torch.zeros(warm.size, dtype=torch.uint8), _CpuKeys(warm))
    sk.insertions_seen += int(st[2])
    PD.sharded_cm_apply(sk, ops, keys)
    return sk.counters.numpy(), sk.increment_counts.numpy(), sk.insertions_seen


def test_sharded_cm_apply_warm_sketch_cross_shard_deletes(oracle):
    """deletes whose inserts live in another shard (or in the
    sketch already) must not raise; the result equals one in-order apply."""
    out = run2(_sharded_cm_fake)
    warm, ops, keys = _warm_stream(11)
    o = oracle.OracleSketch("cm", 4, 64, master_seed=3)
    o.apply_ops(np.zeros(warm.size, np.uint8), warm)
    o.apply_ops(ops, keys)
    a, b = PD.shard_range(ops.size, 1, 2)
    assert (ops[a:b] == 1).sum() > 100
    for r in (0, 1):
        np.testing.assert_array_equal(out[r][0], o.slim)
        np.testing.assert_array_equal(out[r][1], o.inc)
        assert out[r][2] == o.seen


def _sharded_cm_phantom(rank, world):
    sk = _CpuCm(4, 64, 3)
    ops = np.array([0, 0, 0, 1, 1, 0, 1, 0], np.uint8)
    keys = np.array([5, 6, 7, 5, 99, 8, 6, 9], np.uint64)  # key 99 was never inserted
    try:
        PD.sharded_cm_apply(sk, ops, keys)
    except Exception as e:  # noqa: BLE001
        return type(e).__name__, str(e), sk.counters.numpy(), sk.insertions_seen
    return "no error", "", sk.counters.numpy(), sk.insertions_seen


def test_sharded_cm_apply_failure_raises_the_same_error_on_every_rank(oracle):
    """the fallback must raise on every rank (not only rank 0),
    with the reference's message and the state of the ops before the failing
    one."""
    out = run2(_sharded_cm_phantom)
    assert out[0][0] == out[1][0] == "PhantomDeletionError"
    assert out[0][1] == out[1][1] and "op 4" in out[0][1] and "99" in out[0][1]
    o = oracle.OracleSketch("cm", 4, 64, master_seed=3)
    st = o.apply_ops(np.array([0, 0, 0, 1, 1, 0, 1, 0], np.uint8), np.array([5, 6, 7, 5, 99, 8, 6, 9], np.uint64))
    assert st[0] == 1
    for r in (0, 1):
        np.testing.assert_array_equal(out[r][2], o.slim)
        assert out[r][3] == o.seen == 3
