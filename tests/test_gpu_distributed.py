"""World-size-2 runs of the multi-GPU paths through the real GPU API (gloo
process group over CUDA tensors; both ranks share the one GPU of the test
box, and no kernel of one rank waits on the other's): sharded count-min
builds (``CmSketch.sharded_apply_`` = ``distributed.sharded_cm_apply``:
global precheck, raw signed deltas from ``sfk_cm_delta``, one sum
all-reduce) on a warm sketch with cross-shard deletes, the exact fallback
with a phantom delete (same exception on every rank), and the query layout
of north_star: build on rank 0, ``broadcast_slim_``, each rank answers a
contiguous slice. Each result is compared with one single-process
``apply_ops`` / ``query_many`` (and the CPU oracle)."""

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, fn, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    except Exception as e:  # noqa: BLE001
        q.put((rank, ("worker error", repr(e))))
    finally:
        dist.destroy_process_group()


def run2(fn):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, fn, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    return out


def _cm_stream(seed, n_keys=5000, n_warm=200_000, n_ins=400_000, n_del=200_000):
    rng = np.random.default_rng(seed)
    keys = rng.integers(0, 1 << 62, size=n_keys, dtype=np.uint64)
    warm = rng.choice(keys, size=n_warm)
    ops = np.concatenate([np.zeros(n_ins, np.uint8), np.ones(n_del, np.uint8)])
    ks = np.concatenate([rng.choice(keys, size=n_ins), rng.choice(warm, size=n_del)])
    perm = rng.permutation(ops.size)
    return warm, ops[perm], ks[perm]


def _gpu_sharded_cm(rank, world):
    import paper_1701_04148_b200 as P

    warm, ops, keys = _cm_stream(21)
    cm = P.CmSketch(P.SketchParams(d=4, w=4096, master_seed=9))
    cm.apply_ops(np.zeros(warm.size, np.uint8), warm)
    cm.sharded_apply_(torch.from_numpy(ops).cuda(), torch.from_numpy(keys).cuda())
    return cm.counters.cpu().numpy(), cm.increment_counts.cpu().numpy(), cm.insertions_seen


def test_sharded_cm_apply_gpu_warm_cross_shard_deletes(oracle):
    import paper_1701_04148_b200 as P
    from paper_1701_04148_b200 import distributed as PD

    out = run2(_gpu_sharded_cm)
    warm, ops, keys = _cm_stream(21)
    a, b = PD.shard_range(ops.size, 1, 2)
    assert (ops[a:b] == 1).sum() > 50_000
    cm = P.CmSketch(P.SketchParams(d=4, w=4096, master_seed=9))
    cm.apply_ops(np.zeros(warm.size, np.uint8), warm)
    cm.apply_ops(ops, keys)
    o = oracle.OracleSketch("cm", 4, 4096, master_seed=9)
    o.apply_ops(np.zeros(warm.size, np.uint8), warm)
    o.apply_ops(ops, keys)
    np.testing.assert_array_equal(cm.counters.cpu().numpy(), o.slim)
    for r in (0, 1):
        assert not isinstance(out[r][0], str), out[r]
        np.testing.assert_array_equal(out[r][0], o.slim)
        np.testing.assert_array_equal(out[r][1], o.inc)
        assert out[r][2] == o.seen == cm.insertions_seen


def _gpu_sharded_cm_phantom(rank, world):
    import paper_1701_04148_b200 as P

    rng = np.random.default_rng(4)
    keys = rng.integers(0, 1 << 40, size=100_000, dtype=np.uint64)
    ops = np.zeros(keys.size, np.uint8)
    ops[70_000] = 1
    keys[70_000] = 12345  # never inserted: the first failing op
    cm = P.CmSketch(P.SketchParams(d=4, w=1 << 20, master_seed=1))
    try:
        cm.sharded_apply_(ops, keys)
    except Exception as e:  # noqa: BLE001
        return type(e).__name__, str(e), cm.counters.cpu().numpy(), cm.insertions_seen
    return "no error", "", cm.counters.cpu().numpy(), cm.insertions_seen


def test_sharded_cm_apply_gpu_fallback_raises_on_every_rank(oracle):
    out = run2(_gpu_sharded_cm_phantom)
    rng = np.random.default_rng(4)
    keys = rng.integers(0, 1 << 40, size=100_000, dtype=np.uint64)
    ops = np.zeros(keys.size, np.uint8)
    ops[70_000] = 1
    keys[70_000] = 12345
    o = oracle.OracleSketch("cm", 4, 1 << 20, master_seed=1)
    st = o.apply_ops(ops, keys)
    assert st[0] == 1 and st[1] == 70_000
    assert out[0][0] == out[1][0] == "PhantomDeletionError", out
    assert out[0][1] == out[1][1] and "op 70000" in out[0][1]
    for r in (0, 1):
        np.testing.assert_array_equal(out[r][2], o.slim)
        assert out[r][3] == o.seen == 70_000


def _gpu_bcast_query(rank, world):
    import paper_1701_04148_b200 as P
    from paper_1701_04148_b200 import distributed as PD, workloads as W

    c = W.cfg3(seed=6, n_ins=500_000, v=50_000, alpha=1.0)
    sk = P.SfSketch(P.SketchParams(d=4, w=65536, z=4, master_seed=6), "sff")
    if rank == 0:
        sk.apply_ops(c["ops"], c["keys"])
    sk.broadcast_slim_(src=0)
    q = torch.from_numpy(W.query_keys(8, c["distinct"], 1.0, 0, 3_000_001)).cuda()
    est, a, b = PD.sharded_query(sk, q)
    return est.cpu().numpy(), a, b


def test_broadcast_slim_then_sharded_queries_equal_one_gpu(oracle):
    import paper_1701_04148_b200 as P
    from paper_1701_04148_b200 import workloads as W

    out = run2(_gpu_bcast_query)
    c = W.cfg3(seed=6, n_ins=500_000, v=50_000, alpha=1.0)
    sk = P.SfSketch(P.SketchParams(d=4, w=65536, z=4, master_seed=6), "sff")
    sk.apply_ops(c["ops"], c["keys"])
    q = W.query_keys(8, c["distinct"], 1.0, 0, 3_000_001)
    want = sk.query_many(torch.from_numpy(q).cuda()).cpu().numpy()
    got = np.concatenate([out[0][0], out[1][0]])
    assert out[0][1] == 0 and out[0][2] == out[1][1] and out[1][2] == q.size
    np.testing.assert_array_equal(got, want)
    o = oracle.OracleSketch("sff", 4, 65536, 4, None, 6)
    o.apply_ops(c["ops"], c["keys"].astype(np.uint64))
    np.testing.assert_array_equal(got[:300_000], o.query_many(q[:300_000].astype(np.uint64)))
