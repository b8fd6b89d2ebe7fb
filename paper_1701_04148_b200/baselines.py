"""The four baseline sketches on the GPU (drop-in for ``CmSketch``,
``CountSketch``, ``CuSketch`` and ``CmlSketch`` of ``sfsketch.baselines``,
``baselines.py:46-238``).

* ``CmSketch.apply_ops``: when no op of the batch can fail (checked on the
  device from the counter extremes and the batch's insert/delete counts),
  one pass of warp-aggregated atomics applies it; otherwise an exact
  sort + prefix-scan pass finds the first failing op and applies exactly the
  ops before it. ``allreduce_`` merges stream-sharded builds (NCCL sum).
* ``CuSketch.apply_ops``: the ordered dataflow engine with an unbounded cap
  (every insert raises its minimal counters), or the exact sequential device
  engine if the batch could reach a saturated minimum.
* ``CountSketch``: signed +-1 per row; one pass of warp-aggregated atomics
  when no counter can reach +-2^31 within the batch, else the sequential
  engine. Query: the reference's signed median, in registers.
* ``CmlSketch``: the ordered engine with each insert's coin flip turned into
  a cap on the minimum exponent (``base ** -c`` tabulated on the host with
  the same libm ``pow`` the reference's numba kernel calls). Query: the min
  exponent decoded through a table of the reference's ``cml_value``.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from ._ops import OP_DELETE, OP_INSERT, Scratch, device, normalize_stream, raise_for_status, single_op
import math

from .errors import ConfigurationError, UnsupportedOperationError
from .hashing import MASK64, seed_array
from .params import SketchParams
from .sf import query_min, query_min_host


class _CounterSketch:
    kind = ""
    supports_deletion = True
    _device_checks_ops = False
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
        # CM / CU validate op codes on the device (status BAD_OPCODE)
        ops_t, kb = normalize_stream(ops, keys, check_ops=not self._device_checks_ops, stage=self._scratch)
        result = self._submit(ops_t, kb, sequential)
        status, bad, n_ins = Scratch.read(result, self._scratch)
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

    def query_many_host(self, keys, out=None):
        """Host keys in, host int64 estimates out (``sfk_min_query_host``)."""
        res = query_min_host(self.counters, self._seeds, keys, out)
        return res if isinstance(keys, torch.Tensor) or out is not None else res.numpy()


class CmSketch(_CounterSketch):
    """Count-min: +1 per row on insert, -1 on delete; query = row minimum."""

    kind = "cm"
    supports_deletion = True
    _entry = "sfk_cm_apply"
    _ws_entry = "sfk_cm_workspace_size"
    _device_checks_ops = True

    def allreduce_(self, group=None) -> None:
        """Merge stream-sharded replicas in place: counters and tallies are
        sums over shards (count-min updates commute). uint32 counters travel
        as int32; two's-complement sums wrap exactly like uint32 sums, and a
        merged counter above 2^32 - 1 raises ``SaturationError`` on every
        rank."""
        from .distributed import allreduce_counters_

        self.insertions_seen = allreduce_counters_(self.counters, self.increment_counts, self.insertions_seen, group)

    def sharded_apply_(self, ops, keys, group=None) -> None:
        """``apply_ops`` over a batch every rank holds, computed by all ranks
        together (``distributed.sharded_cm_apply``)."""
        from .distributed import sharded_cm_apply

        sharded_cm_apply(self, ops, keys, group)

    # hooks of distributed.sharded_cm_apply
    _normalize = staticmethod(normalize_stream)
    _raise_for_status = staticmethod(raise_for_status)

    def _cm_delta_(self, delta: torch.Tensor, ops_t: torch.Tensor, kb) -> None:
        """Raw signed +-1 per row into `delta` (mod 2^32, no checks)."""
        L = _lib.lib()
        p = self.params
        _lib.check(L.sfk_cm_delta(delta.data_ptr(), self._seeds.ctypes.data, p.d, p.w, ops_t.data_ptr(), kb.ptr(),
                                  kb.kind, kb.rec_len, kb.n, _lib.stream_ptr()), "sfk_cm_delta")


class CuSketch(_CounterSketch):
    """Conservative update: +1 only to the hashed counters equal to the
    minimum. Not reversible, so deletion is unsupported."""

    kind = "cu"
    supports_deletion = False
    _entry = "sfk_cu_apply"
    _ws_entry = "sfk_cu_workspace_size"
    _device_checks_ops = True

    def delete(self, key: int) -> None:
        raise UnsupportedOperationError("conservative update cannot be reversed; deletion is unsupported")


class CountSketch:
    """Signed-median sketch: d arrays of w int32 counters (``baselines.py:90-128``).
    Insert adds a per-row sign, delete subtracts it; query = median of the
    sign-corrected reads (even d: mean of the central pair, half away from
    zero), clamped at zero."""

    kind = "c"
    supports_deletion = True

    def __init__(self, params: SketchParams):
        self.params = params
        self.counters = torch.zeros((params.d, params.w), dtype=torch.int32, device=device())
        self._seeds = seed_array(params.master_seed, 0, params.d)
        self.insertions_seen = 0
        self._scratch = Scratch()

    def insert(self, key: int) -> None:
        self.apply_ops(*single_op(OP_INSERT, key))

    def delete(self, key: int) -> None:
        self.apply_ops(*single_op(OP_DELETE, key))

    def apply_ops(self, ops, keys, *, sequential: bool = False) -> None:
        ops_t, kb = normalize_stream(ops, keys)
        L = _lib.lib()
        p = self.params
        result, ws = self._scratch.get(int(L.sfk_count_workspace_size(p.d, p.w, kb.n)))
        rc = L.sfk_count_apply(self.counters.data_ptr(), self._seeds.ctypes.data, p.d, p.w, ops_t.data_ptr(),
                               kb.ptr(), kb.kind, kb.rec_len, kb.n, result.data_ptr(), ws.data_ptr(), ws.numel(),
                               _lib.FLAG_SEQUENTIAL if sequential else 0, _lib.stream_ptr())
        _lib.check(rc, "sfk_count_apply")
        status, bad, n_ins = Scratch.read(result)
        self.insertions_seen += n_ins
        raise_for_status(status, bad, kb)

    def query(self, key: int) -> int:
        return int(self.query_many(np.array([int(key) & MASK64], dtype=np.uint64))[0].item())

    def query_many(self, keys) -> torch.Tensor:
        return count_query(self.counters, self._seeds, keys)


def count_query(counters: torch.Tensor, seeds: np.ndarray, keys) -> torch.Tensor:
    """``_kernels.count_query`` (``_kernels.py:149-179``) on the GPU."""
    from ._ops import normalize_keys

    kb = normalize_keys(keys)
    d, w = counters.shape
    out = torch.empty(kb.n, dtype=torch.int64, device=counters.device)
    if kb.n:
        rc = _lib.lib().sfk_count_query(counters.data_ptr(), seeds.ctypes.data, d, w, kb.ptr(), kb.kind, kb.rec_len,
                                        kb.n, out.data_ptr(), _lib.stream_ptr())
        _lib.check(rc, "sfk_count_query")
    return out


def cml_value(exponent, base: float):
    """Point value of a log counter (``baselines.py:174-179``), host numpy,
    the reference's formula: round((base**c - 1) / (base - 1)), ties away."""
    c = np.asarray(exponent, dtype=np.float64)
    with np.errstate(over="ignore", invalid="ignore"):
        vals = np.expm1(c * math.log(base)) / (base - 1.0)
        return np.floor(vals + 0.5).astype(np.int64)


_CML_TABLES = {}


def cml_tables(base: float, dev):
    """Device tables for one base: gate[c] = base ** -c (the host libm pow the
    reference's numba kernel calls) and value[c] = cml_value(c, base)."""
    key = (float(base), str(dev))
    if key not in _CML_TABLES:
        b = float(base)
        gate = np.array([b ** -float(c) for c in range(65536)], dtype=np.float64)
        value = cml_value(np.arange(65536), b)
        _CML_TABLES[key] = (torch.from_numpy(gate).to(dev), torch.from_numpy(value).to(dev))
    return _CML_TABLES[key]


def cml_query(exps: torch.Tensor, seeds: np.ndarray, keys, value_table=None) -> torch.Tensor:
    """``_kernels.cml_min_exp`` (``_kernels.py:214-226``), decoded through
    ``value_table`` when given."""
    from ._ops import normalize_keys

    kb = normalize_keys(keys)
    d, w = exps.shape
    out = torch.empty(kb.n, dtype=torch.int64, device=exps.device)
    if kb.n:
        vt = value_table.data_ptr() if value_table is not None else None
        rc = _lib.lib().sfk_cml_query(exps.data_ptr(), seeds.ctypes.data, d, w, kb.ptr(), kb.kind, kb.rec_len, kb.n,
                                      vt, out.data_ptr(), _lib.stream_ptr())
        _lib.check(rc, "sfk_cml_query")
    return out


class CmlSketch:
    """Log-counter sketch: d arrays of w uint16 exponents (``baselines.py:182-238``).
    Insert number n draws u = finalize64(rng_seed + (n+1) GOLDEN) and, with
    probability base ** -c, raises every hashed cell still at the minimum
    exponent c. No deletion."""

    kind = "cml"
    supports_deletion = False
    DEFAULT_BASE = 1.08

    def __init__(self, params: SketchParams, base: float = DEFAULT_BASE, rng_seed=None):
        if not base > 1.0:
            raise ConfigurationError(f"base must be > 1, got {base}")
        self.params = params
        self.base = float(base)
        self.rng_seed = params.master_seed if rng_seed is None else int(rng_seed) & MASK64
        self.exponents = torch.zeros((params.d, params.w), dtype=torch.uint16, device=device())
        self._seeds = seed_array(params.master_seed, 0, params.d)
        self.insertions_seen = 0
        self._scratch = Scratch()

    def insert(self, key: int) -> None:
        self.apply_ops(*single_op(OP_INSERT, key))

    def delete(self, key: int) -> None:
        raise UnsupportedOperationError("log counters cannot be decremented; deletion is unsupported")

    def apply_ops(self, ops, keys, *, sequential: bool = False) -> None:
        ops_t, kb = normalize_stream(ops, keys)
        L = _lib.lib()
        p = self.params
        gate, _ = cml_tables(self.base, self.exponents.device)
        result, ws = self._scratch.get(int(L.sfk_cml_workspace_size(p.d, p.w, kb.n)))
        rc = L.sfk_cml_apply(self.exponents.data_ptr(), self._seeds.ctypes.data, p.d, p.w, ops_t.data_ptr(), kb.ptr(),
                             kb.kind, kb.rec_len, kb.n, gate.data_ptr(), self.rng_seed, self.insertions_seen,
                             result.data_ptr(), ws.data_ptr(), ws.numel(), _lib.FLAG_SEQUENTIAL if sequential else 0,
                             _lib.stream_ptr())
        _lib.check(rc, "sfk_cml_apply")
        status, bad, n_ins = Scratch.read(result)
        self.insertions_seen += n_ins
        raise_for_status(status, bad, kb)

    def query(self, key: int) -> int:
        return int(self.query_many(np.array([int(key) & MASK64], dtype=np.uint64))[0].item())

    def query_many(self, keys) -> torch.Tensor:
        _, value = cml_tables(self.base, self.exponents.device)
        return cml_query(self.exponents, self._seeds, keys, value)
