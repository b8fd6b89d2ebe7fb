"""Count-min and conservative-update baselines on the GPU (drop-in for the
``CmSketch`` / ``CuSketch`` of ``sfsketch.baselines``, ``baselines.py:46-171``).

* ``CmSketch.apply_ops``: when no op of the batch can fail (checked on the
  device from the counter extremes and the batch's insert/delete counts),
  one pass of warp-aggregated atomics applies it; otherwise an exact
  sort + prefix-scan pass finds the first failing op and applies exactly the
  ops before it. ``allreduce_`` merges stream-sharded builds (NCCL sum).
* ``CuSketch.apply_ops``: the ordered dataflow engine with an unbounded cap
  (every insert raises its minimal counters), or the exact sequential device
  engine if the batch could reach a saturated minimum.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from ._ops import OP_DELETE, OP_INSERT, Scratch, device, normalize_stream, raise_for_status, single_op
from .errors import UnsupportedOperationError
from .hashing import MASK64, seed_array
from .params import SketchParams
from .sf import query_min


class _CounterSketch:
    kind = ""
    supports_deletion = True
    _entry = ""
    _ws_entry = ""

    def __init__(self, params: SketchParams):
        self.params = params
        dev = device()
        self.counters = torch.zeros((params.d, params.w), dtype=torch.uint32, device=dev)
        self._seeds = seed_array(params.master_seed, 0, params.d)
        self.increment_counts = torch.zeros(params.d, dtype=torch.int64, device=dev)
        self.insertions_seen = 0
        self._scratch = Scratch()

    def insert(self, key: int) -> None:
        self.apply_ops(*single_op(OP_INSERT, key))

    def delete(self, key: int) -> None:
        self.apply_ops(*single_op(OP_DELETE, key))

    def apply_ops(self, ops, keys, *, sequential: bool = False) -> None:
        ops_t, kb = normalize_stream(ops, keys)
        result = self._submit(ops_t, kb, sequential)
        status, bad, n_ins = Scratch.read(result)
        self.insertions_seen += n_ins
        raise_for_status(status, bad, kb)

    def _submit(self, ops_t, kb, sequential: bool = False) -> torch.Tensor:
        L = _lib.lib()
        p = self.params
        ws_bytes = int(getattr(L, self._ws_entry)(p.d, p.w, kb.n)) if not sequential else 256
        result, ws = self._scratch.get(ws_bytes)
        rc = getattr(L, self._entry)(
            self.counters.data_ptr(), self._seeds.ctypes.data, p.d, p.w, ops_t.data_ptr(), kb.ptr(), kb.kind,
            kb.rec_len, kb.n, self.increment_counts.data_ptr(), result.data_ptr(), ws.data_ptr(), ws.numel(),
            _lib.FLAG_SEQUENTIAL if sequential else 0, _lib.stream_ptr(),
        )
        _lib.check(rc, self._entry)
        return result

    def query(self, key: int) -> int:
        return int(self.query_many(np.array([int(key) & MASK64], dtype=np.uint64))[0].item())

    def query_many(self, keys) -> torch.Tensor:
        return query_min(self.counters, self._seeds, keys)


class CmSketch(_CounterSketch):
    """Count-min: +1 per row on insert, -1 on delete; query = row minimum."""

    kind = "cm"
    supports_deletion = True
    _entry = "sfk_cm_apply"
    _ws_entry = "sfk_cm_workspace_size"

    def allreduce_(self, group=None) -> None:
        """Merge stream-sharded replicas in place: counters and tallies are
        sums over shards (count-min updates commute). uint32 counters travel
        as int32; two's-complement sums wrap exactly like uint32 sums."""
        from .distributed import allreduce_counters_

        self.insertions_seen = allreduce_counters_(self.counters, self.increment_counts, self.insertions_seen, group)


class CuSketch(_CounterSketch):
    """Conservative update: +1 only to the hashed counters equal to the
    minimum. Not reversible, so deletion is unsupported."""

    kind = "cu"
    supports_deletion = False
    _entry = "sfk_cu_apply"
    _ws_entry = "sfk_cu_workspace_size"

    def delete(self, key: int) -> None:
        raise UnsupportedOperationError("conservative update cannot be reversed; deletion is unsupported")
