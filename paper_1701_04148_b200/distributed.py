"""Multi-GPU plumbing for the two paths that shard.

* Point queries: independent per key. The slim is replicated from one rank
  (``broadcast_counters_``, NCCL broadcast over NVLink) and every rank answers
  a contiguous slice of the batch (``shard_range``, ``sharded_query``).
* Count-min builds: updates commute. ``sharded_cm_apply`` replaces one
  ``cm_apply`` call (``_kernels.py:62-88``) over a batch every rank holds:
  a global precheck (one all-reduce of the batch's insert/delete counts, and
  the replicated counters' extremes) proves that no op of the whole batch can
  fail; then rank r adds its contiguous slice as raw signed +-1 increments
  (``sfk_cm_delta``: no per-shard saturation/phantom checks, so a delete whose
  insert sits in another shard is fine) to a zeroed delta, the deltas are
  summed with one all-reduce and added to every replica. uint32 values travel
  as int32: two's-complement sums wrap exactly like uint32 sums, and the
  precheck keeps the true result inside [0, 2^32 - 1], so the merge is
  bit-exact. If the precheck fails, rank 0 applies the batch in stream order
  (the exact path, which finds the first failing op), broadcasts the state
  and the outcome, and every rank raises the same exception.
* ``allreduce_counters_`` merges independently built replicas (sum); it
  raises ``SaturationError`` on every rank if a merged counter would exceed
  2^32 - 1 (the reference never wraps).
* SF and CU updates are order-dependent: replicas only (single-GPU build).

Everything here works on any torch.distributed backend: the bench runs it on
``nccl``; the tests run it on ``gloo`` with CPU tensors (a CPU stand-in
sketch) and with CUDA tensors through the real GPU sketch.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from .errors import SaturationError

U32MAX = 0xFFFFFFFF


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous slice [a, b) of n items owned by `rank`."""
    per = n // world
    a = rank * per
    b = n if rank == world - 1 else a + per
    return a, b


def _extremes(counters: torch.Tensor) -> torch.Tensor:
    """[max, min] of uint32 counters as an int64 device tensor (no host sync)."""
    if counters.numel() == 0:
        return torch.zeros(2, dtype=torch.int64, device=counters.device)
    # flipping the sign bit maps uint32 order onto int32 order
    s = counters.view(torch.int32) ^ torch.tensor(-(1 << 31), dtype=torch.int32, device=counters.device)
    mn, mx = torch.aminmax(s)
    return torch.stack([mx, mn]).to(torch.int64) + (1 << 31)


def allreduce_counters_(counters: torch.Tensor, tallies: torch.Tensor | None = None, seen: int = 0,
                        group=None) -> int:
    """Sum uint32 counters (and int64 tallies, and the insert count) over
    ranks in place; returns the global insertions_seen. Raises
    ``SaturationError`` on every rank when a merged counter would exceed
    2^32 - 1: the sum of the ranks' maxima bounds every merged counter, and
    only when that bound fails are the exact sums checked (int64 all-reduce)."""
    dev = counters.device
    head = torch.cat([_extremes(counters)[:1], torch.tensor([int(seen)], dtype=torch.int64, device=dev)])
    dist.all_reduce(head, op=dist.ReduceOp.SUM, group=group)
    max_sum, seen_sum = (int(v) for v in head.tolist())
    if max_sum > U32MAX:
        exact = counters.to(torch.int64)
        dist.all_reduce(exact, op=dist.ReduceOp.SUM, group=group)
        if bool((exact > U32MAX).any()):
            raise SaturationError("merged counter exceeds 2^32 - 1: the shards cannot be summed without wrapping")
    dist.all_reduce(counters.view(torch.int32), op=dist.ReduceOp.SUM, group=group)
    if tallies is not None:
        dist.all_reduce(tallies, op=dist.ReduceOp.SUM, group=group)
    return seen_sum


def broadcast_counters_(counters: torch.Tensor, src: int = 0, group=None) -> None:
    """Replicate uint32 counters from rank `src`."""
    dist.broadcast(counters.view(torch.int32), src=src, group=group)


def _failure_free(n_ins: int, n_del: int, cmax: int, cmin: int) -> bool:
    # sfk_cm_apply's precheck: no insert can meet a saturated counter and no
    # delete a zero one, whatever the order
    return cmax + n_ins <= U32MAX and (n_del == 0 or cmin >= n_del)


def _batch_stats(counters: torch.Tensor, ops_shard: torch.Tensor, group=None) -> list[int]:
    """[global inserts, global deletes, max counter, min counter] with one
    all-reduce and one host read."""
    dev = counters.device
    o = ops_shard.to(dev)
    n_del = (o != 0).sum().to(torch.int64)
    cnt = torch.stack([torch.tensor(int(o.numel()), dtype=torch.int64, device=dev) - n_del, n_del])
    dist.all_reduce(cnt, op=dist.ReduceOp.SUM, group=group)
    return [int(v) for v in torch.cat([cnt, _extremes(counters)]).tolist()]


def batch_is_failure_free(counters: torch.Tensor, ops_shard: torch.Tensor, group=None) -> bool:
    """Global form of the CM precheck over every rank's shard of the batch."""
    return _failure_free(*_batch_stats(counters, ops_shard, group))


def sharded_cm_apply(sketch, ops, keys, group=None) -> None:
    """``sketch.apply_ops(ops, keys)`` for a replicated count-min sketch,
    computed by all ranks together (every rank passes the same full batch).

    The sketch supplies ``_normalize(ops, keys) -> (ops_t, kb)``,
    ``_cm_delta_(delta, ops_t, kb)`` (raw signed +-1 into `delta`) and
    ``_submit(ops_t, kb) -> result`` (the exact in-order apply, returning the
    {status, op_index, n_ins} triple); ``CmSketch`` implements them on the
    GPU."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    ops_t, kb = sketch._normalize(ops, keys)
    n = kb.n
    a, b = shard_range(n, rank, world)
    n_ins, n_del, cmax, cmin = _batch_stats(sketch.counters, ops_t[a:b], group)
    if sketch.params.d <= 8 and _failure_free(n_ins, n_del, cmax, cmin):
        delta = torch.zeros_like(sketch.counters)
        if b > a:
            sketch._cm_delta_(delta, ops_t[a:b], kb.slice(a, b))
        dist.all_reduce(delta.view(torch.int32), op=dist.ReduceOp.SUM, group=group)
        sketch.counters.view(torch.int32).add_(delta.view(torch.int32))
        sketch.increment_counts.add_(n_ins)
        sketch.insertions_seen += n_ins
        return
    # exact fallback: rank 0 applies in stream order; every rank receives the
    # state and the outcome, and raises the same exception
    dev = sketch.counters.device
    outcome = torch.zeros(3, dtype=torch.int64, device=dev)
    if rank == 0:
        outcome.copy_(sketch._submit(ops_t, kb))
    broadcast_counters_(sketch.counters, 0, group)
    dist.broadcast(sketch.increment_counts, src=0, group=group)
    dist.broadcast(outcome, src=0, group=group)
    status, bad, done = (int(v) for v in outcome.tolist())
    sketch.insertions_seen += done
    sketch._raise_for_status(status, bad, kb)


def sharded_query(sketch, keys, group=None):
    """This rank's contiguous slice of ``sketch.query_many(keys)`` (the slim
    replicated beforehand, e.g. with ``broadcast_slim_``); returns
    (estimates, a, b) with the slice bounds."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n = int(keys.shape[0]) if hasattr(keys, "shape") else len(keys)
    a, b = shard_range(n, rank, world)
    return sketch.query_many(keys[a:b]), a, b
