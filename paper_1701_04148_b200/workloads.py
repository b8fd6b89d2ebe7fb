"""Seeded synthetic streams for the BASELINE.json configurations.

SURVEY.md §8(d): every stream derives from one seed through numpy's PCG64;
Zipf ranks come from the CDF + ``searchsorted`` construction of the
reference generator (``workloads.py:92-103``). The paper's YCSB and campus
traces are absent, so these stand in for them (same shapes, sizes and skew
parameters).

  cfg1  SF1 insert-only: n uint32 keys, Zipf(1.0) over V distinct
  cfg2  CM / CU: n uint32 keys, Zipf(1.0) over V distinct
  cfg3  SFF: n inserts Zipf(alpha) + 20% of the insert occurrences deleted,
        each delete at a uniform random position after its own insert
  cfg4  SF1 on 13-byte records (random 5-tuples), Zipf(1.2)
  cfg5  point queries: half present keys (Zipf(alpha_q) over the present
        set, alpha_q = 0 is uniform), half absent random uint32 — built by a
        counter-based generator so any slice can be regenerated exactly on
        host or device (``query_keys``)
"""

from __future__ import annotations

import numpy as np

from .hashing import GOLDEN, MASK64


def rng_for(seed: int, stream: int = 0) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64([seed, stream]))


def distinct_u32(rng: np.random.Generator, v: int) -> np.ndarray:
    """v distinct random uint32 values, in draw order."""
    out = np.empty(0, dtype=np.uint32)
    while out.shape[0] < v:
        draw = rng.integers(0, 1 << 32, size=int((v - out.shape[0]) * 1.1) + 1024, dtype=np.uint64).astype(np.uint32)
        allv = np.concatenate([out, draw])
        _, first = np.unique(allv, return_index=True)
        out = allv[np.sort(first)]
    return np.ascontiguousarray(out[:v])


def zipf_cdf(v: int, alpha: float) -> np.ndarray:
    w = 1.0 / np.power(np.arange(1, v + 1, dtype=np.float64), alpha)
    cdf = np.cumsum(w / w.sum())
    cdf[-1] = 1.0
    return cdf


def zipf_ranks(rng: np.random.Generator, v: int, alpha: float, n: int, chunk: int = 1 << 24) -> np.ndarray:
    """n ranks in [0, v): Zipf(alpha) (alpha = 0 gives uniform)."""
    if alpha == 0.0:
        return rng.integers(0, v, size=n, dtype=np.int64)
    cdf = zipf_cdf(v, alpha)
    out = np.empty(n, dtype=np.int64)
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        out[a:b] = np.searchsorted(cdf, rng.random(b - a), side="right")
    np.minimum(out, v - 1, out=out)
    return out


def cfg1(seed: int = 2017, n: int = 1_000_000, v: int = 100_000, alpha: float = 1.0) -> dict:
    rng = rng_for(seed, 1)
    distinct = distinct_u32(rng, v)
    keys = distinct[zipf_ranks(rng, v, alpha, n)]
    return {"ops": np.zeros(n, dtype=np.uint8), "keys": keys, "distinct": distinct}


def cfg2(seed: int = 2017, n: int = 10_000_000, v: int = 1_000_000, alpha: float = 1.0) -> dict:
    rng = rng_for(seed, 2)
    distinct = distinct_u32(rng, v)
    keys = distinct[zipf_ranks(rng, v, alpha, n)]
    return {"ops": np.zeros(n, dtype=np.uint8), "keys": keys, "distinct": distinct}


def cfg3(seed: int = 2017, n_ins: int = 10_000_000, v: int = 1_000_000, alpha: float = 1.0,
         del_frac: float = 0.2) -> dict:
    rng = rng_for(seed, 3)
    distinct = distinct_u32(rng, v)
    ins_keys = distinct[zipf_ranks(rng, v, alpha, n_ins)]
    n_del = int(round(n_ins * del_frac))
    victims = rng.choice(n_ins, size=n_del, replace=False)
    u = rng.random(n_del)
    # delete of occurrence p lands strictly after it: position in (p, n_ins]
    dpos = victims + (1.0 - u) * (n_ins - victims)
    pos = np.concatenate([np.arange(n_ins, dtype=np.float64), dpos])
    order = np.argsort(pos, kind="stable")
    ops = np.concatenate([np.zeros(n_ins, np.uint8), np.ones(n_del, np.uint8)])[order]
    keys = np.concatenate([ins_keys, ins_keys[victims]])[order]
    return {"ops": np.ascontiguousarray(ops), "keys": np.ascontiguousarray(keys), "distinct": distinct}


def cfg4(seed: int = 2017, n: int = 100_000_000, v: int = 10_000_000, alpha: float = 1.2, rec_len: int = 13) -> dict:
    rng = rng_for(seed, 4)
    records = rng.integers(0, 256, size=(v, rec_len), dtype=np.uint8)
    ranks = zipf_ranks(rng, v, alpha, n)
    return {"ops": np.zeros(n, dtype=np.uint8), "records": np.ascontiguousarray(records[ranks]),
            "distinct": records}


# ---------------------------------------------------------------- cfg5 queries
def _mix_np(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


class DeviceQueryStream:
    """The cfg-5 query stream generated on the GPU (``sfk_gen_query_keys``):
    ``keys(t0, n)`` equals ``query_keys(seed, present, alpha_q, t0, t0 + n)``."""

    def __init__(self, seed: int, present: np.ndarray, alpha_q: float):
        import torch

        from . import _lib

        self._lib = _lib
        self.seed = int(seed) & MASK64
        dev = torch.device("cuda", torch.cuda.current_device())
        self.present = torch.from_numpy(np.ascontiguousarray(present, dtype=np.uint32)).to(dev)
        self.sorted = torch.from_numpy(np.sort(present).astype(np.uint32)).to(dev)
        self.v = int(present.shape[0])
        self.cdf = None if alpha_q == 0.0 else torch.from_numpy(zipf_cdf(self.v, alpha_q)).to(dev)

    def keys(self, t0: int, n: int, out=None):
        import torch

        if out is None:
            out = torch.empty(n, dtype=torch.uint32, device=self.present.device)
        L = self._lib.lib()
        rc = L.sfk_gen_query_keys(self.seed, self.present.data_ptr(), self.sorted.data_ptr(), self.v,
                                  self.cdf.data_ptr() if self.cdf is not None else None, int(t0), int(n),
                                  out.data_ptr(), self._lib.stream_ptr())
        self._lib.check(rc, "sfk_gen_query_keys")
        return out


def query_keys(seed: int, present: np.ndarray, alpha_q: float, t0: int, t1: int) -> np.ndarray:
    """Keys t0..t1-1 of the cfg-5 query stream (counter-based, so any slice
    is reproducible). Draw t: h = finalize64(seed + (t+1)*GOLDEN); bit 0 picks
    present/absent; present keys take Zipf(alpha_q) rank u = (h >> 11)/2^53 over
    ``present``; absent keys are finalize64(h ^ j*GOLDEN) truncated to 32 bits
    for the first j = 1, 2, ... that is not in ``present``."""
    t = np.arange(t0, t1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        h = _mix_np(np.uint64(seed & MASK64) + (t + np.uint64(1)) * np.uint64(GOLDEN))
    is_present = (h & np.uint64(1)) == 0
    u = (h >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    v = present.shape[0]
    if alpha_q == 0.0:
        ranks = np.minimum((u * v).astype(np.int64), v - 1)
    else:
        ranks = np.minimum(np.searchsorted(zipf_cdf(v, alpha_q), u, side="right"), v - 1)
    out = present[ranks].astype(np.uint32)
    sorted_present = np.sort(present)
    todo = np.nonzero(~is_present)[0]
    j = 1
    while todo.size:
        with np.errstate(over="ignore"):
            cand = (_mix_np(h[todo] ^ (np.uint64(j) * np.uint64(GOLDEN))) & np.uint64(0xFFFFFFFF)).astype(np.uint32)
        pos = np.minimum(np.searchsorted(sorted_present, cand), v - 1)
        hit = sorted_present[pos] == cand
        out[todo[~hit]] = cand[~hit]
        todo = todo[hit]
        j += 1
    return out
