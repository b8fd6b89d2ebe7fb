"""Direct access to the hash kernels (``_kernels.mix_batch`` and the key
loaders) on CUDA tensors; used to pin the device hash family against the
reference goldens."""

from __future__ import annotations

import torch

from . import _lib
from ._ops import normalize_keys


def mix_batch(keys) -> torch.Tensor:
    """finalize64 of every key (``_kernels.py:56-59``); uint64 CUDA tensor."""
    L = _lib.lib()
    kb = normalize_keys(keys)
    if kb.kind != _lib.KEY_U64:
        kb = normalize_keys(load_keys(kb))
    out = torch.empty(kb.n, dtype=torch.uint64, device=kb.tensor.device)
    if kb.n:
        _lib.check(L.sfk_mix_batch(kb.ptr(), kb.n, out.data_ptr(), _lib.stream_ptr()), "sfk_mix_batch")
    return out


def load_keys(keys) -> torch.Tensor:
    """Materialise the u64 key of every element (records hashed with
    FNV-1a-64 + finalize64, ``hashing.py:124-129``)."""
    L = _lib.lib()
    kb = normalize_keys(keys)
    out = torch.empty(kb.n, dtype=torch.uint64, device=kb.tensor.device)
    if kb.n:
        _lib.check(L.sfk_load_keys(kb.ptr(), kb.kind, kb.rec_len, kb.n, out.data_ptr(), _lib.stream_ptr()),
                   "sfk_load_keys")
    return out
