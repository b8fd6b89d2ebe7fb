"""Multi-GPU plumbing for the two paths that shard.

* Point queries: independent per key. The slim is replicated from one rank
  (``broadcast_counters_``, NCCL broadcast over NVLink) and every rank answers
  a contiguous slice of the batch (``shard_range``).
* Count-min builds: updates commute, so each rank applies a contiguous slice
  of the stream to a zero-initialised replica and the replicas are summed
  (``allreduce_counters_``, one NCCL all-reduce). uint32 counters travel as
  int32: two's-complement sums wrap exactly like uint32 sums, so the merge is
  bit-exact. Sharding changes where a failing op would be detected, so
  ``sharded_cm_apply`` first checks globally (one all-reduce of the counter
  extremes and op counts) that no op of the batch can fail; otherwise it
  applies the batch on one rank, in stream order, and broadcasts.
* SF and CU updates are order-dependent: replicas only (single-GPU build).

Everything here works on any torch.distributed backend; the tests run it on
``gloo`` with CPU tensors, the bench on ``nccl`` with CUDA tensors.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous slice [a, b) of n items owned by `rank`."""
    per = n // world
    a = rank * per
    b = n if rank == world - 1 else a + per
    return a, b


def allreduce_counters_(counters: torch.Tensor, tallies: torch.Tensor | None = None, seen: int = 0,
                        group=None) -> int:
    """Sum uint32 counters (and int64 tallies, and the insert count) over
    ranks in place; returns the global insertions_seen."""
    dist.all_reduce(counters.view(torch.int32), op=dist.ReduceOp.SUM, group=group)
    if tallies is not None:
        dist.all_reduce(tallies, op=dist.ReduceOp.SUM, group=group)
    s = torch.tensor([int(seen)], dtype=torch.int64, device=counters.device)
    dist.all_reduce(s, op=dist.ReduceOp.SUM, group=group)
    return int(s.item())


def broadcast_counters_(counters: torch.Tensor, src: int = 0, group=None) -> None:
    """Replicate uint32 counters from rank `src`."""
    dist.broadcast(counters.view(torch.int32), src=src, group=group)


def batch_is_failure_free(counters: torch.Tensor, ops_shard: torch.Tensor, group=None) -> bool:
    """Global form of the CM precheck: no insert of the batch can meet a
    saturated counter (max + total inserts <= 2^32 - 1) and no delete a zero
    one (total deletes == 0 or min >= total deletes)."""
    dev = counters.device
    c64 = counters.to(torch.int64)
    n_del = int((ops_shard != 0).sum().item())
    n_ins = int(ops_shard.numel()) - n_del
    cnt = torch.tensor([n_ins, n_del], dtype=torch.int64, device=dev)
    dist.all_reduce(cnt, op=dist.ReduceOp.SUM, group=group)
    cmax = int(c64.max().item()) if c64.numel() else 0
    cmin = int(c64.min().item()) if c64.numel() else 0
    tot_ins, tot_del = (int(v) for v in cnt.tolist())
    return cmax + tot_ins <= 0xFFFFFFFF and (tot_del == 0 or cmin >= tot_del)


def sharded_cm_apply(sketch, ops, keys, group=None) -> None:
    """Apply one stream to a replicated ``CmSketch`` with every rank holding the
    full stream: rank r applies slice r to a zeroed delta replica, the deltas
    are summed and added. The result equals ``sketch.apply_ops(ops, keys)`` on
    one GPU (falls back to exactly that, on rank 0 + broadcast, when an op of
    the batch could fail)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    ops_t = torch.as_tensor(ops)
    n = int(ops_t.shape[0])
    if not batch_is_failure_free(sketch.counters, ops_t[slice(*shard_range(n, rank, world))].to(
            sketch.counters.device), group):
        err = None
        if rank == 0:
            try:
                sketch.apply_ops(ops, keys)
            except Exception as e:  # noqa: BLE001 - re-raised on every rank below
                err = e
        broadcast_counters_(sketch.counters, 0, group)
        dist.broadcast(sketch.increment_counts, src=0, group=group)
        seen = torch.tensor([sketch.insertions_seen], dtype=torch.int64, device=sketch.counters.device)
        dist.broadcast(seen, src=0, group=group)
        sketch.insertions_seen = int(seen.item())
        if err is not None:
            raise err
        return
    a, b = shard_range(n, rank, world)
    delta = type(sketch)(sketch.params)
    delta.apply_ops(ops[a:b], keys[a:b])
    seen = allreduce_counters_(delta.counters, delta.increment_counts, delta.insertions_seen, group)
    sketch.counters.view(torch.int32).add_(delta.counters.view(torch.int32))
    sketch.increment_counts.add_(delta.increment_counts)
    sketch.insertions_seen += seen
