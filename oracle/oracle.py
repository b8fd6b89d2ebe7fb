"""TEST INFRASTRUCTURE ONLY — ctypes front end of the CPU oracle.

The oracle is a plain-C restatement (``sfsketch_oracle.c``) of the reference's
sequential numba kernels (``/root/reference/pkg/src/sfsketch/_kernels.py``).
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this module, and only as the checker or as the timed CPU
baseline; the product package ``paper_1701_04148_b200`` never imports it.

Every function mirrors one reference kernel and takes/returns numpy arrays
with the reference's dtypes. Apply functions mutate their state arrays in
place and return ``(status, op_index, n_ins)`` like the reference
(``_kernels.py:1-16``).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

OK, PHANTOM, SATURATED, UNSUPPORTED = 0, 1, 2, 3

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I = ctypes.c_int


def build() -> str:
    """Compile the oracle with its Makefile (gcc, seconds)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.orc_mix_batch.argtypes = [_P, _I64, _P]
        L.orc_seed_for_index.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        L.orc_seed_for_index.restype = ctypes.c_uint64
        L.orc_keys_from_records.argtypes = [_P, _I64, _I64, _P]
        L.orc_min_query.argtypes = [_P, _P, _I, _I64, _P, _I64, _P]
        L.orc_min_query_mt.argtypes = [_P, _P, _I, _I64, _P, _I, _I64, _P, _I]
        L.orc_max_threads.restype = _I
        for name in ("orc_cm_apply", "orc_cu_apply"):
            f = getattr(L, name)
            f.argtypes = [_P, _P, _I, _I64, _P, _P, _I64, _P, _P, _P]
            f.restype = _I
        L.orc_sf_flat_apply.argtypes = [_P, _P, _P, _P, _P, _I, _I64, _I64, _I, _P, _P, _I64, _P, _P, _P]
        L.orc_sf_flat_apply.restype = _I
        L.orc_sf_bucket_apply.argtypes = [_P, _P, _P, _P, _I, _I64, _I64, _I, _P, _P, _I64, _P, _P, _P]
        L.orc_sf_bucket_apply.restype = _I
        L.orc_oracle_slim_apply.argtypes = [_P, _P, _I, _I64, _P, _P, _I64, _P, _P, _P]
        L.orc_oracle_slim_apply.restype = _I
        L.orc_count_apply.argtypes = [_P, _P, _I, _I64, _P, _P, _I64, _P, _P]
        L.orc_count_apply.restype = _I
        L.orc_count_query.argtypes = [_P, _P, _I, _I64, _P, _I64, _P]
        L.orc_cml_apply.argtypes = [_P, _P, _I, _I64, _P, _P, _I64, ctypes.c_double, ctypes.c_uint64, _I64, _P, _P]
        L.orc_cml_apply.restype = _I
        L.orc_cml_min_exp.argtypes = [_P, _P, _I, _I64, _P, _I64, _P]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    assert a.flags.c_contiguous, "oracle arrays must be C-contiguous"
    return a.ctypes.data


def _u64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint64)


def _u8(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint8)


# ---------------------------------------------------------------- hashing
def finalize64(x: int) -> int:
    """hashing.py:33-45 (scalar, pure Python)."""
    m = 0xFFFFFFFFFFFFFFFF
    x &= m
    x ^= x >> 30
    x = (x * 0xBF58476D1CE4E5B9) & m
    x ^= x >> 27
    x = (x * 0x94D049BB133111EB) & m
    x ^= x >> 31
    return x


def mix_batch(keys) -> np.ndarray:
    """_kernels.py:56-59."""
    keys = _u64(keys)
    out = np.empty_like(keys)
    lib().orc_mix_batch(_ptr(keys), keys.shape[0], _ptr(out))
    return out


def seed_array(master: int, start: int, count: int) -> np.ndarray:
    """hashing.py:132-137."""
    return np.array([lib().orc_seed_for_index(master, start + i) for i in range(count)], dtype=np.uint64)


def keys_from_records(recs: np.ndarray) -> np.ndarray:
    """FNV-1a-64 + finalize64 over fixed-size byte records (hashing.py:124-129)."""
    recs = np.ascontiguousarray(recs, dtype=np.uint8)
    n, rec = recs.shape
    out = np.empty(n, dtype=np.uint64)
    lib().orc_keys_from_records(_ptr(recs), n, rec, _ptr(out))
    return out


# ---------------------------------------------------------------- query
def min_query(counters: np.ndarray, seeds: np.ndarray, keys, threads: int = 1, out=None) -> np.ndarray:
    """_kernels.py:229-241; ``threads > 1`` splits keys like bench.py:153-162.
    ``out`` (int64, len(keys)) may be passed to avoid page-faulting a fresh array."""
    counters = np.ascontiguousarray(counters, dtype=np.uint32)
    seeds = _u64(seeds)
    keys = np.ascontiguousarray(keys)
    if keys.dtype == np.uint32:
        key32 = 1
    else:
        keys = _u64(keys)
        key32 = 0
    d, w = counters.shape
    if out is None:
        out = np.empty(keys.shape[0], dtype=np.int64)
    if threads == 1 and not key32:
        lib().orc_min_query(_ptr(counters), _ptr(seeds), d, w, _ptr(keys), keys.shape[0], _ptr(out))
    else:
        lib().orc_min_query_mt(_ptr(counters), _ptr(seeds), d, w, _ptr(keys), key32, keys.shape[0], _ptr(out), threads)
    return out


def max_threads() -> int:
    return int(lib().orc_max_threads())


# ---------------------------------------------------------------- apply
def _apply_tail(status, op_index, n_ins):
    return int(status), int(op_index.value), int(n_ins.value)


def cm_apply(counters, seeds, ops, keys, inc_counts):
    """_kernels.py:62-88 (mutates counters, inc_counts)."""
    ops, keys, seeds = _u8(ops), _u64(keys), _u64(seeds)
    d, w = counters.shape
    oi, ni = _I64(), _I64()
    st = lib().orc_cm_apply(_ptr(counters), _ptr(seeds), d, w, _ptr(ops), _ptr(keys), ops.shape[0],
                            _ptr(inc_counts), ctypes.byref(oi), ctypes.byref(ni))
    return _apply_tail(st, oi, ni)


def cu_apply(counters, seeds, ops, keys, inc_counts):
    """_kernels.py:91-115 (mutates counters, inc_counts)."""
    ops, keys, seeds = _u8(ops), _u64(keys), _u64(seeds)
    d, w = counters.shape
    oi, ni = _I64(), _I64()
    st = lib().orc_cu_apply(_ptr(counters), _ptr(seeds), d, w, _ptr(ops), _ptr(keys), ops.shape[0],
                            _ptr(inc_counts), ctypes.byref(oi), ctypes.byref(ni))
    return _apply_tail(st, oi, ni)


def sf_flat_apply(slim, fat, dsub, slim_seeds, fat_seeds, variant, ops, keys, inc_counts):
    """_kernels.py:244-315 (variants 1, 2, 3)."""
    ops, keys = _u8(ops), _u64(keys)
    slim_seeds, fat_seeds = _u64(slim_seeds), _u64(fat_seeds)
    d, w = slim.shape
    wp = fat.shape[1]
    oi, ni = _I64(), _I64()
    dptr = _ptr(dsub) if dsub is not None else None
    st = lib().orc_sf_flat_apply(_ptr(slim), _ptr(fat), dptr, _ptr(slim_seeds), _ptr(fat_seeds), d, w, wp,
                                 int(variant), _ptr(ops), _ptr(keys), ops.shape[0], _ptr(inc_counts),
                                 ctypes.byref(oi), ctypes.byref(ni))
    return _apply_tail(st, oi, ni)


def sf_bucket_apply(slim, fat, bucket_seeds, slot_seeds, mode, ops, keys, inc_counts):
    """_kernels.py:318-384 (mode 0 sum trigger, 1 max clamp, 2 changed-max)."""
    ops, keys = _u8(ops), _u64(keys)
    bucket_seeds, slot_seeds = _u64(bucket_seeds), _u64(slot_seeds)
    d, w, z = fat.shape
    oi, ni = _I64(), _I64()
    st = lib().orc_sf_bucket_apply(_ptr(slim), _ptr(fat), _ptr(bucket_seeds), _ptr(slot_seeds), d, w, z,
                                   int(mode), _ptr(ops), _ptr(keys), ops.shape[0], _ptr(inc_counts),
                                   ctypes.byref(oi), ctypes.byref(ni))
    return _apply_tail(st, oi, ni)


def oracle_slim_apply(slim, seeds, keys, true_counts, inc_counts):
    """_kernels.py:387-411."""
    keys, seeds = _u64(keys), _u64(seeds)
    true_counts = np.ascontiguousarray(true_counts, dtype=np.int64)
    d, w = slim.shape
    oi, ni = _I64(), _I64()
    st = lib().orc_oracle_slim_apply(_ptr(slim), _ptr(seeds), d, w, _ptr(keys), _ptr(true_counts),
                                     keys.shape[0], _ptr(inc_counts), ctypes.byref(oi), ctypes.byref(ni))
    return _apply_tail(st, oi, ni)


def count_apply(counters, seeds, ops, keys):
    """_kernels.py:118-146 (mutates the int32 counters)."""
    ops, keys, seeds = _u8(ops), _u64(keys), _u64(seeds)
    d, w = counters.shape
    oi, ni = _I64(), _I64()
    st = lib().orc_count_apply(_ptr(counters), _ptr(seeds), d, w, _ptr(ops), _ptr(keys), ops.shape[0],
                               ctypes.byref(oi), ctypes.byref(ni))
    return _apply_tail(st, oi, ni)


def count_query(counters, seeds, keys) -> np.ndarray:
    """_kernels.py:149-179."""
    keys, seeds = _u64(keys), _u64(seeds)
    d, w = counters.shape
    out = np.empty(keys.shape[0], dtype=np.int64)
    lib().orc_count_query(_ptr(counters), _ptr(seeds), d, w, _ptr(keys), keys.shape[0], _ptr(out))
    return out


def cml_apply(exps, seeds, ops, keys, base, rng_seed, start_pos):
    """_kernels.py:182-211 (mutates the uint16 exponents)."""
    ops, keys, seeds = _u8(ops), _u64(keys), _u64(seeds)
    d, w = exps.shape
    oi, ni = _I64(), _I64()
    st = lib().orc_cml_apply(_ptr(exps), _ptr(seeds), d, w, _ptr(ops), _ptr(keys), ops.shape[0], float(base),
                             int(rng_seed) & 0xFFFFFFFFFFFFFFFF, int(start_pos), ctypes.byref(oi), ctypes.byref(ni))
    return _apply_tail(st, oi, ni)


def cml_min_exp(exps, seeds, keys) -> np.ndarray:
    """_kernels.py:214-226."""
    keys, seeds = _u64(keys), _u64(seeds)
    d, w = exps.shape
    out = np.empty(keys.shape[0], dtype=np.int64)
    lib().orc_cml_min_exp(_ptr(exps), _ptr(seeds), d, w, _ptr(keys), keys.shape[0], _ptr(out))
    return out


def cml_value(exponent, base: float) -> np.ndarray:
    """baselines.py:174-179: round((base**c - 1) / (base - 1)), ties away from zero."""
    import math

    c = np.asarray(exponent, dtype=np.float64)
    vals = np.expm1(c * math.log(base)) / (base - 1.0)
    return np.floor(vals + 0.5).astype(np.int64)


class OracleSketch:
    """Whole-sketch state mirroring ``SfSketch`` / ``CmSketch`` / ``CuSketch``
    (sf.py:105-193, baselines.py:46-171) on numpy arrays, driven by the
    oracle kernels above. Used as the parity reference in tests and as the
    CPU baseline in bench.py."""

    def __init__(self, kind: str, d: int, w: int, z: int = 1, w_prime=None, master_seed: int = 0):
        self.kind = kind
        self.d, self.w, self.z = d, w, z
        self.w_prime = z * w if w_prime is None else w_prime
        self.master_seed = master_seed
        self.slim_seeds = seed_array(master_seed, 0, d)
        self.ext_seeds = seed_array(master_seed, d, d)
        self.slim = np.zeros((d, w), dtype=np.uint32)
        self.inc = np.zeros(d, dtype=np.int64)
        self.seen = 0
        self.fat = None
        self.dsub = None
        if kind in ("sf1", "sf2"):
            self.fat = np.zeros((d, self.w_prime), dtype=np.uint32)
            self.fat_seeds = self.ext_seeds
            if kind == "sf2":
                self.dsub = np.zeros((d, w), dtype=np.uint32)
        elif kind == "sf3":
            self.fat = np.zeros((d, z * w), dtype=np.uint32)
            self.fat_seeds = self.slim_seeds
        elif kind in ("sf4", "sff"):
            self.fat = np.zeros((d, w, z), dtype=np.uint32)
            self.fat_seeds = self.ext_seeds

    def apply_ops(self, ops, keys):
        if self.kind == "cm":
            r = cm_apply(self.slim, self.slim_seeds, ops, keys, self.inc)
        elif self.kind == "cu":
            r = cu_apply(self.slim, self.slim_seeds, ops, keys, self.inc)
        elif self.kind in ("sf1", "sf2", "sf3"):
            code = {"sf1": 1, "sf2": 2, "sf3": 3}[self.kind]
            r = sf_flat_apply(self.slim, self.fat, self.dsub, self.slim_seeds, self.fat_seeds, code, ops, keys, self.inc)
        else:
            mode = 0 if self.kind == "sf4" else 1
            r = sf_bucket_apply(self.slim, self.fat, self.slim_seeds, self.fat_seeds, mode, ops, keys, self.inc)
        self.seen += r[2]
        return r

    def query_many(self, keys, threads: int = 1, out=None):
        return min_query(self.slim, self.slim_seeds, keys, threads, out)
