"""Slim-fat sketch family on the GPU (drop-in for ``sfsketch.sf``).

Same classes, attributes and methods as the reference (``sf.py:50-258``);
state lives in CUDA tensors and every update/query runs in the sm_100a
kernels behind ``libsfsketch_cuda.so``:

  SF1  flat fat (d, w'); no deletion           -> parallel engine (max-raise runs)
  SF2  flat fat + deletion sub-sketch          -> parallel engine (sum trigger, op-by-op runs)
  SF3  flat fat of width z*w folded onto w     -> parallel engine (sum trigger, fold groups as buckets)
  SF4  bucketed fat (d, w, z), sum trigger     -> parallel engine (sum trigger)
  SFF  bucketed fat (d, w, z), max clamp       -> parallel engine (max clamp)

  (d > 8, z > 8, or ``sequential=True`` use the exact one-thread device engine)

Attributes tests read (``slim.counters``, ``slim.increment_counts``,
``slim.insertions_seen``, ``fat.counters``, ``deletion_sub.counters``,
``params``, ``variant``, ``kind``) keep their names; counters are torch
``uint32`` CUDA tensors (``.cpu().numpy()`` gives the reference's numpy
view). ``query_many`` returns an int64 CUDA tensor.
"""

from __future__ import annotations

from enum import Enum

import numpy as np
import torch

from . import _lib
from ._ops import (
    OP_DELETE,
    OP_INSERT,
    Scratch,
    device,
    normalize_host_keys,
    normalize_keys,
    normalize_stream,
    raise_for_status,
    single_op,
)
from .errors import ConfigurationError, UnsupportedOperationError
from .hashing import MASK64, seed_array
from .params import SketchParams


class Variant(str, Enum):
    SF1 = "sf1"
    SF2 = "sf2"
    SF3 = "sf3"
    SF4 = "sf4"
    SFF = "sff"


def _zeros(shape) -> torch.Tensor:
    return torch.zeros(shape, dtype=torch.uint32, device=device())


class SlimSubsketch:
    """Query-side (d, w) counters plus per-row raise tallies."""

    __slots__ = ("counters", "increment_counts", "insertions_seen")

    def __init__(self, d: int, w: int):
        self.counters = _zeros((d, w))
        self.increment_counts = torch.zeros(d, dtype=torch.int64, device=device())
        self.insertions_seen = 0


class FatSubsketchFlat:
    __slots__ = ("counters",)

    def __init__(self, counters: torch.Tensor):
        self.counters = counters


class FatSubsketchBucketed:
    __slots__ = ("counters",)

    def __init__(self, counters: torch.Tensor):
        self.counters = counters


class DeletionSubsketch:
    __slots__ = ("counters",)

    def __init__(self, counters: torch.Tensor):
        self.counters = counters


def query_min(counters: torch.Tensor, seeds: np.ndarray, keys) -> torch.Tensor:
    """Fused hash + d gathers + min on the GPU (``_kernels.min_query``)."""
    L = _lib.lib()
    kb = normalize_keys(keys)
    d, w = counters.shape
    out = torch.empty(kb.n, dtype=torch.int64, device=counters.device)
    if kb.n:
        rc = L.sfk_min_query(counters.data_ptr(), seeds.ctypes.data, d, w, kb.ptr(), kb.kind, kb.rec_len, kb.n,
                             out.data_ptr(), _lib.stream_ptr())
        _lib.check(rc, "sfk_min_query")
    return out


class StagedKeys:
    """A device copy of a host key batch's first ``n`` keys, uploaded on a
    side stream (``stage_query_keys``) so the copy can overlap a build."""

    __slots__ = ("buf", "n", "kind", "rec_len", "event", "_src", "_alloc")

    def __init__(self, buf, n, kind, rec_len, src):
        self.buf, self.n, self.kind, self.rec_len, self.event, self._src = buf, n, kind, rec_len, None, src
        self._alloc = torch.cuda.Event()  # the buffer's allocation is ordered on the current stream
        self._alloc.record(torch.cuda.current_stream(buf.device))

    def issue(self) -> None:
        """Enqueue the copy on the side stream (once)."""
        if self.event is not None:
            return
        dev = self.buf.device
        side = _stage_streams.get(dev.index)
        if side is None:
            side = _stage_streams[dev.index] = torch.cuda.Stream(dev)
        side.wait_event(self._alloc)  # not on later work of the current stream (the build it overlaps)
        with torch.cuda.stream(side):
            self.buf.copy_(self._src, non_blocking=True)
        self.buf.record_stream(side)
        self.event = torch.cuda.Event()
        self.event.record(side)
        self._src = None


_stage_streams: dict = {}


def stage_query_keys(keys_host, count: int | None = None, *, defer: bool = False) -> StagedKeys:
    """Start copying the first ``count`` keys (default: all) of a host batch
    to the device on a side stream and return at once. Pass the handle with
    the SAME host batch to ``query_min_host(..., staged=...)``: its chunks
    inside the staged prefix are then queried in place, with no H2D on the
    query's critical path (``sfk_min_query_host_staged``). Pinned host keys
    make the copy asynchronous. ``defer=True`` only prepares the handle: the
    copy starts at ``handle.issue()`` (``SfSketch.stage_query_keys`` issues it
    inside the next ``apply_ops``, after that batch's own upload), or at the
    query at the latest."""
    t, kind, rec, n = normalize_host_keys(keys_host)
    m = n if count is None else max(0, min(int(count), n))
    flat = t.view(torch.uint8).reshape(-1)
    esz = flat.numel() // n if n else 1
    h = StagedKeys(torch.empty(m * esz, dtype=torch.uint8, device=device()), m, kind, rec, flat[: m * esz])
    if not defer:
        h.issue()
    return h


def query_min_host(counters: torch.Tensor, seeds: np.ndarray, keys_host, out_host: torch.Tensor | None = None,
                   staged: StagedKeys | None = None):
    """Point queries for a batch that lives in HOST memory (pinned or
    pageable), the reference's ``query_many`` contract (``sf.py:189-193``):
    host keys in, host int64 estimates out. ``sfk_min_query_host`` cuts the
    batch into chunks that flow H2D -> fused hash/gather/min kernel -> D2H on
    three streams, as in the paper's GPU query design,
    with the estimates narrowed on the link and widened into ``out_host`` by
    native host threads. ``out_host`` (int64 CPU tensor, same length) is
    allocated when omitted; returns it."""
    L = _lib.lib()
    t, kind, rec, n = normalize_host_keys(keys_host)
    if out_host is None:
        out_host = torch.empty(n, dtype=torch.int64)
    elif (out_host.device.type != "cpu" or out_host.dtype != torch.int64 or tuple(out_host.shape) != (n,)
          or not out_host.is_contiguous()):
        raise ConfigurationError("out_host must be a contiguous int64 CPU tensor of the batch's length")
    d, w = counters.shape
    if staged is not None and (staged.kind != kind or staged.rec_len != rec or staged.n > n):
        raise ConfigurationError("staged keys do not match this batch's key type or length")
    if n:
        if staged is not None and staged.n:
            staged.issue()
            torch.cuda.current_stream(device()).wait_event(staged.event)
            rc = L.sfk_min_query_host_staged(counters.data_ptr(), seeds.ctypes.data, d, w, t.data_ptr(), kind, rec,
                                             n, out_host.data_ptr(), staged.buf.data_ptr(), staged.n,
                                             _lib.stream_ptr())
        else:
            rc = L.sfk_min_query_host(counters.data_ptr(), seeds.ctypes.data, d, w, t.data_ptr(), kind, rec, n,
                                      out_host.data_ptr(), _lib.stream_ptr())
        _lib.check(rc, "sfk_min_query_host")
    return out_host


class SfSketch:
    """One of the five slim-fat variants over a shared interface."""

    supports_deletion = True  # except SF1, which raises

    def __init__(self, params: SketchParams, variant):
        self.variant = Variant(variant)
        self.params = params
        d, w, z = params.d, params.w, params.z
        if d > 64:
            raise ConfigurationError("d > 64 is not supported by the GPU kernels")
        self.slim = SlimSubsketch(d, w)
        self._slim_seeds = seed_array(params.master_seed, 0, d)
        self._ext_seeds = seed_array(params.master_seed, d, d)
        self.deletion_sub = None
        if self.variant in (Variant.SF1, Variant.SF2):
            self.fat = FatSubsketchFlat(_zeros((d, params.w_prime)))
            self._fat_seeds = self._ext_seeds
            if self.variant is Variant.SF2:
                self.deletion_sub = DeletionSubsketch(_zeros((d, w)))
        elif self.variant is Variant.SF3:
            if params.w_prime != z * w:
                raise ConfigurationError(
                    f"the fold variant needs w_prime == z*w, got w_prime={params.w_prime}, z*w={z * w}"
                )
            self.fat = FatSubsketchFlat(_zeros((d, z * w)))
            self._fat_seeds = self._slim_seeds
        else:
            self.fat = FatSubsketchBucketed(_zeros((d, w, z)))
            self._fat_seeds = self._ext_seeds
        self._used_normal = False
        self._used_oracle = False
        self._scratch = Scratch()
        self._deferred_stage: list = []

    @property
    def kind(self) -> str:
        return self.variant.value

    # ------------------------------------------------------------ updates
    def insert(self, key: int) -> None:
        self.apply_ops(*single_op(OP_INSERT, key))

    def delete(self, key: int) -> None:
        if self.variant is Variant.SF1:
            raise UnsupportedOperationError("this variant has no deletion path")
        self.apply_ops(*single_op(OP_DELETE, key))

    def apply_ops(self, ops, keys, *, sequential: bool = False) -> None:
        """Replay a batch in stream order (``sf.py:149-184``).

        ``sequential=True`` runs the exact one-thread device engine instead of
        the parallel one (a cross-check; both produce identical state)."""
        if self._used_oracle:
            raise UnsupportedOperationError(
                "sketch already ran in oracle-assisted mode; regular updates would break it"
            )
        # op codes checked on the device; small host batches read in place from pinned staging
        ops_t, kb = normalize_stream(ops, keys, check_ops=False, stage=self._scratch)
        result = self._submit(ops_t, kb, sequential)
        while self._deferred_stage:  # query keys staged to upload behind this batch's own
            self._deferred_stage.pop().issue()
        status, bad, n_ins = Scratch.read(result, self._scratch)
        if kb.n and status != _lib.BAD_OPCODE:  # a rejected batch leaves the sketch untouched
            self._used_normal = True
        self.slim.insertions_seen += n_ins
        raise_for_status(status, bad, kb)

    def _submit(self, ops_t: torch.Tensor, kb, sequential: bool = False) -> torch.Tensor:
        """Enqueue the apply on the current stream; returns the device result
        triple {status, op_index, n_ins} without synchronising."""
        L = _lib.lib()
        p = self.params
        code = _lib.VARIANT_CODE[self.variant.value]
        wp = p.w_prime if self.variant in (Variant.SF1, Variant.SF2, Variant.SF3) else 0
        if self.variant is Variant.SF3:
            wp = p.z * p.w
        ws_bytes = int(L.sfk_sf_workspace_size(code, p.d, p.w, wp, p.z, kb.n)) if not sequential else 256
        result, ws = self._scratch.get(ws_bytes)
        dsub = self.deletion_sub.counters.data_ptr() if self.deletion_sub is not None else None
        rc = L.sfk_sf_apply(
            code, self.slim.counters.data_ptr(), self.fat.counters.data_ptr(), dsub,
            self._slim_seeds.ctypes.data, self._fat_seeds.ctypes.data, p.d, p.w, wp, p.z,
            ops_t.data_ptr(), kb.ptr(), kb.kind, kb.rec_len, kb.n,
            self.slim.increment_counts.data_ptr(), result.data_ptr(), ws.data_ptr(), ws.numel(),
            _lib.FLAG_SEQUENTIAL if sequential else 0, _lib.stream_ptr(),
        )
        _lib.check(rc, "sfk_sf_apply")
        return result

    # ------------------------------------------------------------ queries
    def query(self, key: int) -> int:
        return int(self.query_many(np.array([int(key) & MASK64], dtype=np.uint64))[0].item())

    def query_many(self, keys) -> torch.Tensor:
        return query_min(self.slim.counters, self._slim_seeds, keys)

    def stage_query_keys(self, keys, count: int | None = None, *, with_next_apply: bool = False) -> StagedKeys:
        """Upload a prefix of a host query batch before the sketch is final;
        see ``stage_query_keys``. ``with_next_apply=True`` starts the copy
        inside the next ``apply_ops``, right after that batch's upload, so it
        overlaps the build instead of delaying it."""
        h = stage_query_keys(keys, count, defer=with_next_apply)
        if with_next_apply:
            self._deferred_stage.append(h)
        return h

    def query_many_host(self, keys, out=None, staged: StagedKeys | None = None):
        """``query_many`` for host-resident keys with host-resident results
        (the reference's numpy-in / numpy-out form): a numpy array for array or
        list input, else the int64 CPU tensor ``out`` (allocated if omitted).
        ``staged``: a ``stage_query_keys`` handle for a prefix of ``keys``."""
        res = query_min_host(self.slim.counters, self._slim_seeds, keys, out, staged)
        return res if isinstance(keys, torch.Tensor) or out is not None else res.numpy()

    # ------------------------------------------------------------ oracle mode
    def oracle_assisted_insert(self, key: int, true_freq: int) -> None:
        self.oracle_assisted_apply(
            np.array([int(key) & MASK64], dtype=np.uint64), np.array([true_freq], dtype=np.int64)
        )

    def oracle_assisted_apply(self, keys, true_counts, *, sequential: bool = False) -> None:
        """Slim updates gated by exact post-insert counts (``sf.py:199-229``):
        the ordered engine with the true count as each op's cap (op-by-op
        replay), or the exact sequential engine when ``sequential`` or a count
        exceeds 2^32 - 1."""
        if self._used_normal:
            raise UnsupportedOperationError(
                "sketch already saw normal updates; oracle-assisted inserts would break it"
            )
        kb = normalize_keys(keys)
        tc = torch.as_tensor(np.ascontiguousarray(true_counts, dtype=np.int64)) if not isinstance(
            true_counts, torch.Tensor) else true_counts.to(torch.int64)
        if tuple(tc.shape) != (kb.n,):
            raise ConfigurationError("true_counts must match keys in length")
        tc = tc.to(device()).contiguous()
        if kb.n:
            self._used_oracle = True
        L = _lib.lib()
        p = self.params
        ws_bytes = int(L.sfk_oracle_workspace_size(p.d, p.w, kb.n)) if not sequential else 256
        result, ws = self._scratch.get(ws_bytes)
        rc = L.sfk_oracle_slim_apply(
            self.slim.counters.data_ptr(), self._slim_seeds.ctypes.data, p.d, p.w, kb.ptr(), kb.kind, kb.rec_len,
            tc.data_ptr(), kb.n, self.slim.increment_counts.data_ptr(), result.data_ptr(), ws.data_ptr(), ws.numel(),
            _lib.FLAG_SEQUENTIAL if sequential else 0, _lib.stream_ptr(),
        )
        _lib.check(rc, "sfk_oracle_slim_apply")
        status, bad, n_ins = Scratch.read(result)
        self.slim.insertions_seen += n_ins
        raise_for_status(status, bad, kb)

    # ------------------------------------------------------------ export / checks
    def export_slim(self) -> bytes:
        from .serialize import export_slim

        return export_slim(self)

    def check_invariants(self) -> None:
        """Per-variant structural invariants (``sf.py:237-258``), on device."""
        a = self.slim.counters.to(torch.int64)
        fat = self.fat.counters.to(torch.int64)
        if self.variant is Variant.SFF:
            assert bool((a <= fat.amax(dim=2)).all()), "slim counter exceeds its fat bucket max"
        elif self.variant is Variant.SF4:
            assert bool((a <= fat.sum(dim=2)).all()), "slim counter exceeds its fat bucket sum"
        elif self.variant is Variant.SF3:
            d, w, z = self.params.d, self.params.w, self.params.z
            assert bool((a <= fat.reshape(d, z, w).sum(dim=1)).all()), "slim counter exceeds its associated fat sum"
        elif self.variant is Variant.SF2:
            assert bool((a <= self.deletion_sub.counters.to(torch.int64)).all()), (
                "slim counter exceeds its deletion-subsketch bound"
            )

    # ------------------------------------------------------------ multi-GPU
    def broadcast_slim_(self, src: int = 0, group=None) -> None:
        """Replicate the query side from rank ``src`` (NCCL broadcast over
        NVLink; the uint32 counters travel as their int32 bit pattern)."""
        from .distributed import broadcast_counters_

        broadcast_counters_(self.slim.counters, src=src, group=group)
