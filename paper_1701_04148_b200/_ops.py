"""Batch normalisation and status mapping (drop-in for ``sfsketch._ops``).

The reference casts keys to contiguous uint64 and ops to uint8 in {0, 1}
(``_ops.py:20-34``) and maps kernel status codes to exceptions
(``_ops.py:44-59``). Here batches become CUDA tensors that the C ABI reads in
place:

* ``uint32`` keys stay 4 bytes wide and are zero-extended on the device
  (bit-identical to the reference's cast, half the bytes to move);
* signed or narrower integer keys are widened to int64 and reinterpreted as
  uint64 exactly as numpy's cast does;
* a 2-d ``uint8`` array of shape (n, rec_len) is a batch of fixed-size byte
  records, hashed on the device with FNV-1a-64 + finalize64
  (``hashing.key_from_string`` for the same bytes).
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import (
    ConfigurationError,
    PhantomDeletionError,
    SaturationError,
    UnsupportedOperationError,
)
from .hashing import MASK64, key_from_bytes

OP_INSERT = 0
OP_DELETE = 1


def device() -> torch.device:
    _lib.lib()  # fail loudly without CUDA / the built library
    return torch.device("cuda", torch._C._cuda_getDevice())


@dataclass
class KeyBatch:
    tensor: torch.Tensor  # CUDA, contiguous
    kind: int
    rec_len: int
    n: int

    def ptr(self) -> int:
        return self.tensor.data_ptr()

    def key_at(self, t: int) -> int:
        v = self.tensor[t].cpu()
        if self.kind == _lib.KEY_RECORD:
            return key_from_bytes(bytes(v.numpy().tobytes()))
        if self.kind == _lib.KEY_U32:
            return int(v.item())
        return int(v.view(torch.int64).item()) & MASK64

    def slice(self, a: int, b: int) -> "KeyBatch":
        return KeyBatch(self.tensor[a:b], self.kind, self.rec_len, b - a)


def _host_view(arr: np.ndarray) -> torch.Tensor:
    """Zero-copy tensor over a host array that is only read (copied to the
    device); read-only arrays (np.frombuffer, memmaps) are accepted as-is."""
    if arr.flags.writeable:
        return torch.from_numpy(arr)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", UserWarning)
        return torch.from_numpy(arr)


def _to_device(t: torch.Tensor, dev: torch.device) -> torch.Tensor:
    if t.device != dev:
        t = t.to(dev, non_blocking=t.is_pinned())
    return t.contiguous()


def normalize_keys(keys) -> KeyBatch:
    dev = device()
    if isinstance(keys, KeyBatch):
        return keys
    if not isinstance(keys, torch.Tensor):
        arr = np.asarray(keys)
        if arr.dtype == object or arr.dtype.kind not in "iub":
            arr = np.ascontiguousarray(keys, dtype=np.uint64)
        if arr.dtype.kind == "b":
            arr = arr.astype(np.uint64)
        keys = _host_view(np.ascontiguousarray(arr))
    t = keys
    if t.dtype == torch.uint8 and t.dim() == 2:
        t = _to_device(t, dev)
        return KeyBatch(t, _lib.KEY_RECORD, int(t.shape[1]), int(t.shape[0]))
    if t.dim() != 1:
        raise ConfigurationError("keys must be a 1-d sequence")
    if t.dtype == torch.uint32:
        return KeyBatch(_to_device(t, dev), _lib.KEY_U32, 0, int(t.shape[0]))
    if t.dtype == torch.uint64:
        return KeyBatch(_to_device(t, dev), _lib.KEY_U64, 0, int(t.shape[0]))
    if t.dtype == torch.int64:
        return KeyBatch(_to_device(t, dev).view(torch.uint64), _lib.KEY_U64, 0, int(t.shape[0]))
    if t.dtype in (torch.int32, torch.int16, torch.int8, torch.uint8, torch.uint16, torch.bool):
        w = _to_device(t, dev).to(torch.int64)
        return KeyBatch(w.view(torch.uint64), _lib.KEY_U64, 0, int(t.shape[0]))
    raise ConfigurationError(f"keys must be integers, got {t.dtype}")


def normalize_host_keys(keys):
    """``normalize_keys`` for a batch that stays in host memory (the
    host-buffer query path): returns (contiguous CPU tensor, key kind,
    rec_len, n) with the same dtype rules and errors, and no device copy."""
    if isinstance(keys, KeyBatch):
        raise ConfigurationError("host queries take host keys, not a device KeyBatch")
    if isinstance(keys, torch.Tensor):
        if keys.device.type != "cpu":
            raise ConfigurationError("host queries take keys in host memory")
        t = keys
    else:
        arr = np.asarray(keys)
        if arr.dtype == object or arr.dtype.kind not in "iub":
            arr = np.ascontiguousarray(keys, dtype=np.uint64)
        if arr.dtype.kind == "b":
            arr = arr.astype(np.uint64)
        t = _host_view(np.ascontiguousarray(arr))
    if t.dtype == torch.uint8 and t.dim() == 2:
        t = t.contiguous()
        return t, _lib.KEY_RECORD, int(t.shape[1]), int(t.shape[0])
    if t.dim() != 1:
        raise ConfigurationError("keys must be a 1-d sequence")
    if t.dtype == torch.uint32:
        return t.contiguous(), _lib.KEY_U32, 0, int(t.shape[0])
    if t.dtype in (torch.uint64, torch.int64):
        return t.contiguous().view(torch.uint64), _lib.KEY_U64, 0, int(t.shape[0])
    if t.dtype in (torch.int32, torch.int16, torch.int8, torch.uint8, torch.uint16, torch.bool):
        return t.to(torch.int64).view(torch.uint64), _lib.KEY_U64, 0, int(t.shape[0])
    raise ConfigurationError(f"keys must be integers, got {t.dtype}")


BAD_OPCODE_MSG = "op codes must be 0 (insert) or 1 (delete)"


def normalize_stream(ops, keys, check_ops: bool = True, stage: "Scratch | None" = None):
    """``_ops.py:27-34``. ``check_ops=False``: the op codes are validated on
    the device by the apply itself (SF, CM, CU: status BAD_OPCODE, nothing
    applied, raised as the same ConfigurationError by raise_for_status), which
    saves a reduction and a host sync per batch. ``stage``: the caller's
    Scratch, for an apply that synchronises before it returns; a small HOST
    batch is then copied into its pinned staging area, which the kernels read
    in place through its device mapping (no copy launches)."""
    if stage is not None:
        st = stage.stage_host(ops, keys)
        if st is not None:
            o, kb = st
            if check_ops and kb.n and bool((o > OP_DELETE).any()):
                raise ConfigurationError(BAD_OPCODE_MSG)
            return o, kb
    dev = device()
    kb = normalize_keys(keys)
    if isinstance(ops, torch.Tensor):
        o = ops
    else:
        o = _host_view(np.ascontiguousarray(ops, dtype=np.uint8))
    if o.dim() != 1 or int(o.shape[0]) != kb.n:
        raise ConfigurationError("ops and keys must be 1-d sequences of equal length")
    if o.dtype != torch.uint8:
        o = o.to(torch.uint8) if o.device == dev else o.to(torch.uint8)
    o = _to_device(o, dev)
    if check_ops and kb.n and bool((o > OP_DELETE).any()):
        raise ConfigurationError(BAD_OPCODE_MSG)
    return o, kb


def single_op(op_code: int, key: int):
    return (
        np.array([op_code], dtype=np.uint8),
        np.array([int(key) & MASK64], dtype=np.uint64),
    )


def raise_for_status(status: int, op_index: int, keys: KeyBatch) -> None:
    """``_ops.py:44-59``: the same exception types and messages."""
    if status == _lib.OK:
        return
    if status == _lib.BAD_OPCODE:
        raise ConfigurationError(BAD_OPCODE_MSG)
    key = keys.key_at(op_index)
    if status == _lib.PHANTOM:
        raise PhantomDeletionError(f"op {op_index}: deleting key {key} would drive a counter below zero")
    if status == _lib.SATURATED:
        raise SaturationError(f"op {op_index}: counter for key {key} is saturated")
    if status == _lib.UNSUPPORTED:
        raise UnsupportedOperationError(f"op {op_index}: this sketch does not support that operation")
    raise AssertionError(f"unexpected kernel status {status}")


STAGE_MAX_BYTES = 1 << 16  # host batches up to this many key bytes are staged in pinned memory


class Scratch:
    """Per-sketch scratch: the result triple, a growable device workspace and
    a pinned staging area for small host batches.

    The result triple lives in pinned host memory, which the kernels write
    through its (unified-address) device mapping, so reading it back costs a
    stream synchronisation and no copy launch. The staging area is read the
    same way; it is reused by the next apply, which is safe because every
    apply that stages synchronises before it returns."""

    def __init__(self):
        self.result = None
        self.result_np = None
        self.ws = None
        self._dev = None
        self._stage = None
        self._stage_np = None

    def get(self, nbytes: int):
        dev = device()
        if self.result is None or self._dev != dev:
            self.result = torch.zeros(3, dtype=torch.int64).pin_memory()
            self.result_np = self.result.numpy()
            self.ws = None
            self._dev = dev
        if self.ws is None or self.ws.numel() < nbytes:
            self.ws = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=dev)
        return self.result, self.ws

    def stage_host(self, ops, keys):
        """(ops, KeyBatch) over the pinned staging area for a small host batch
        (numpy arrays, sequences or CPU tensors), with the dtype rules of
        normalize_keys; None when the batch is on the device or too large."""
        if isinstance(keys, KeyBatch) or (isinstance(keys, torch.Tensor) and keys.device.type != "cpu"):
            return None
        if isinstance(ops, torch.Tensor) and ops.device.type != "cpu":
            return None
        k = keys.numpy() if isinstance(keys, torch.Tensor) else np.asarray(keys)
        if k.dtype == object or k.dtype.kind not in "iub":
            k = np.asarray(keys, dtype=np.uint64)
        if k.dtype.kind == "b":
            k = k.astype(np.uint64)
        if k.dtype == np.uint8 and k.ndim == 2:
            kind, rec, n = _lib.KEY_RECORD, int(k.shape[1]), int(k.shape[0])
        elif k.ndim != 1:
            return None  # normalize_keys raises the reference's error
        elif k.dtype == np.uint32:
            kind, rec, n = _lib.KEY_U32, 0, int(k.shape[0])
        else:
            k = k.astype(np.int64, copy=False) if k.dtype != np.uint64 else k
            kind, rec, n = _lib.KEY_U64, 0, int(k.shape[0])
        kbytes = n * (rec if kind == _lib.KEY_RECORD else k.dtype.itemsize)
        if n == 0 or kbytes > STAGE_MAX_BYTES:
            return None
        # the reference's cast (np.ascontiguousarray(ops, dtype=np.uint8)), on the caller's object
        o = np.ascontiguousarray(ops.numpy() if isinstance(ops, torch.Tensor) else ops, dtype=np.uint8)
        if o.ndim != 1 or o.shape[0] != n:
            raise ConfigurationError("ops and keys must be 1-d sequences of equal length")
        if self._stage is None:
            self._stage = torch.empty(2 * STAGE_MAX_BYTES + 256, dtype=torch.uint8).pin_memory()
            self._stage_np = self._stage.numpy()
        kb_off = ((n + 255) // 256) * 256
        self._stage_np[:n] = o
        self._stage_np[kb_off:kb_off + kbytes] = np.ascontiguousarray(k).reshape(-1).view(np.uint8)
        ot = self._stage[:n]
        if kind == _lib.KEY_RECORD:
            kt = self._stage[kb_off:kb_off + kbytes].view(n, rec)
        elif kind == _lib.KEY_U32:
            kt = self._stage[kb_off:kb_off + kbytes].view(torch.uint32)
        else:
            kt = self._stage[kb_off:kb_off + kbytes].view(torch.uint64)
        return ot, KeyBatch(kt, kind, rec, n)

    @staticmethod
    def read(result: torch.Tensor, scratch: "Scratch | None" = None):
        if result.is_cuda:
            s, i, n = (int(v) for v in result.tolist())
        else:  # pinned, written by the device: wait for the stream, then read in place
            _lib.check(_lib.load_library().sfk_stream_sync(_lib.stream_ptr()), "sfk_stream_sync")
            r = scratch.result_np if scratch is not None and scratch.result is result else result.numpy()
            s, i, n = int(r[0]), int(r[1]), int(r[2])
        return s, i, n
