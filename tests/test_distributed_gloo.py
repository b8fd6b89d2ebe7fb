"""Multi-process (world_size 2, gloo, CPU) checks of the sharding logic:
contiguous shards, bit-exact uint32 count-min merge through int32 all-reduce
(including wrap-around), slim broadcast, the global failure-free precheck,
and a sharded CM build (oracle replicas per shard + merge) equal to one
sequential build over the whole stream."""

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
    c = torch.from_numpy(rng.integers(0, 1 << 32, size=(4, 64), dtype=np.uint64).astype(np.uint32))
    tallies = torch.tensor([rank + 1] * 4, dtype=torch.int64)
    mine = c.clone()
    seen = PD.allreduce_counters_(c, tallies, seen=10 * (rank + 1))
    return mine.numpy(), c.numpy(), tallies.numpy(), seen


def test_allreduce_uint32_wraps_exactly():
    out = run2(_merge)
    want = (out[0][0].astype(np.uint64) + out[1][0].astype(np.uint64)) & np.uint64(0xFFFFFFFF)
    for r in (0, 1):
        np.testing.assert_array_equal(out[r][1], want.astype(np.uint32))
        np.testing.assert_array_equal(out[r][2], [3, 3, 3, 3])
        assert out[r][3] == 30


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
