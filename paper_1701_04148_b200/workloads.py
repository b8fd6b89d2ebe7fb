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


# ---------------------------------------------------------------- traces
# The reference's trace format (workloads.py:132-184): one "OP,key" line per
# operation, OP in {I, D}, key a base-10 integer in [0, 2^64); blank lines and
# '#' comments are skipped; line numbers are 1-based over all lines.
class Operation:
    """One trace operation: ``op`` is "insert" or "delete"."""

    __slots__ = ("op", "key")

    def __init__(self, op: str, key: int):
        self.op = op
        self.key = key

    def __eq__(self, other):
        return isinstance(other, Operation) and (self.op, self.key) == (other.op, other.key)

    def __repr__(self):
        return f"Operation(op={self.op!r}, key={self.key!r})"


def _trace_line(line: str, lineno: int):
    """The reference's per-line rules (workloads.py:137-155), for the lines
    the device leaves to the host (non-ASCII) and for error messages.
    Returns None for a skipped line, else (op code, key)."""
    from .errors import TraceFormatError

    stripped = line.strip()
    if not stripped or stripped.startswith("#"):
        return None
    parts = stripped.split(",")
    if len(parts) != 2:
        raise TraceFormatError(lineno, f"expected 'OP,key', got {stripped!r}")
    token, key_text = parts[0].strip(), parts[1].strip()
    if token not in ("I", "D"):
        raise TraceFormatError(lineno, f"unknown op token {token!r}")
    try:
        key = int(key_text, 10)
    except ValueError:
        raise TraceFormatError(lineno, f"bad key {key_text!r}") from None
    if not 0 <= key <= MASK64:
        raise TraceFormatError(lineno, f"key {key} out of 64-bit range")
    return (0 if token == "I" else 1), key


def load_trace(path, device=None):
    """Read a whole trace into (ops uint8, keys uint64) CUDA tensors, parsed
    on the GPU (``csrc/sfk_trace.cu``); same results and the same
    ``TraceFormatError`` (line number and message) as the reference's
    ``load_trace``. Lines with non-ASCII bytes (Unicode whitespace or digits,
    which Python's ``str.strip`` / ``int`` accept) are finished on the host."""
    import torch

    from . import _lib
    from ._ops import device as default_device

    dev = device if device is not None else default_device()
    with open(path, "rb") as fh:
        data = fh.read()
    nb = len(data)
    L = _lib.lib()
    host = np.frombuffer(data, dtype=np.uint8) if nb else np.zeros(1, np.uint8)
    text = torch.from_numpy(host.copy()).to(dev)
    cap = nb + 1
    pos = torch.empty(cap, dtype=torch.int64, device=dev)
    status = torch.zeros(cap, dtype=torch.uint8, device=dev)
    lop = torch.zeros(cap, dtype=torch.uint8, device=dev)
    lkey = torch.zeros(cap, dtype=torch.uint64, device=dev)
    ws = torch.empty(int(L.sfk_trace_workspace_size(nb)), dtype=torch.uint8, device=dev)
    info = np.zeros(3, dtype=np.int64)
    _lib.check(L.sfk_trace_parse_lines(text.data_ptr(), nb, pos.data_ptr(), status.data_ptr(), lop.data_ptr(),
                                       lkey.data_ptr(), info.ctypes.data, ws.data_ptr(), ws.numel(),
                                       _lib.stream_ptr()), "sfk_trace_parse_lines")
    nlines, first_err, n_complex = (int(v) for v in info)

    def line_text(i):
        a = int(pos[i].item())
        b = int(pos[i + 1].item()) if i + 1 < nlines else nb
        return data[a:b].decode("utf-8")

    if n_complex:
        # non-ASCII lines: the reference's rules on the host (Unicode
        # whitespace / digits); an error there counts in line order below
        idx = torch.nonzero(status[:nlines] == 6).flatten().tolist()
        for i in idx:
            if first_err >= 0 and i > first_err:
                break
            try:
                r = _trace_line(line_text(i), i + 1)
            except Exception:  # noqa: BLE001 - re-raised in line order below
                first_err = i if first_err < 0 else min(first_err, i)
                break
            if r is None:
                status[i] = 0
            else:
                status[i] = 1
                lop[i] = r[0]
                lkey[i:i + 1].view(torch.int64).fill_(int(np.array([r[1]], np.uint64).view(np.int64)[0]))
    if first_err >= 0:
        _trace_line(line_text(first_err), first_err + 1)  # raises the reference's error
        raise AssertionError("device flagged a trace line the host parser accepts")
    ops = torch.empty(max(nlines, 1), dtype=torch.uint8, device=dev)
    keys = torch.empty(max(nlines, 1), dtype=torch.uint64, device=dev)
    n_out = np.zeros(1, dtype=np.int64)
    _lib.check(L.sfk_trace_compact(status.data_ptr(), lop.data_ptr(), lkey.data_ptr(), nlines, ops.data_ptr(),
                                   keys.data_ptr(), n_out.ctypes.data, ws.data_ptr(), ws.numel(), nb,
                                   _lib.stream_ptr()), "sfk_trace_compact")
    n = int(n_out[0])
    return ops[:n], keys[:n]


def read_trace(path):
    """Stream Operations out of a trace (the reference's generator
    semantics: operations before a bad line are yielded, then it raises)."""
    from .errors import TraceFormatError

    try:
        ops, keys = load_trace(path)
        err = None
    except TraceFormatError as e:  # parse the prefix before the bad line
        err = e
        with open(path, "r", encoding="utf-8") as fh:
            prefix = [ln for _, ln in zip(range(e.line_number - 1), fh)]
        pairs = [r for i, ln in enumerate(prefix, start=1) if (r := _trace_line(ln, i)) is not None]
        ops = np.array([p[0] for p in pairs], dtype=np.uint8)
        keys = np.array([p[1] for p in pairs], dtype=np.uint64)
    ops_h = ops.cpu().numpy() if hasattr(ops, "cpu") else ops
    keys_h = keys.cpu().numpy() if hasattr(keys, "cpu") else keys
    for o, k in zip(ops_h, keys_h):
        yield Operation("insert" if o == 0 else "delete", int(k))
    if err is not None:
        raise err


def write_trace(path, operations) -> None:
    """Write Operations in the trace format (LF line endings)."""
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        for operation in operations:
            fh.write(f"{'I' if operation.op == 'insert' else 'D'},{operation.key}\n")


# ---------------------------------------------------------------- the reference's synthetic streams
# workloads.WorkloadSpec / generate (workloads.py:46-131), drawn on the GPU:
# the same seed gives the same ops / ranks / keys as the reference.
KINDS = ("uniform", "zipf", "trace")
DELETION_MODES = ("none", "reverse_order", "interleaved")


class WorkloadSpec:
    """What to generate (``workloads.py:46-73``), validated the same way."""

    __slots__ = ("kind", "distinct_items", "total_ops", "zipf_skew", "seed", "deletion_mode", "delete_prob",
                 "trace_path")

    def __init__(self, kind, distinct_items=0, total_ops=0, zipf_skew=0.99, seed=0, deletion_mode="none",
                 delete_prob=0.0, trace_path=None):
        from .errors import ConfigurationError

        for name, val in (("kind", kind), ("distinct_items", distinct_items), ("total_ops", total_ops),
                          ("zipf_skew", zipf_skew), ("seed", seed), ("deletion_mode", deletion_mode),
                          ("delete_prob", delete_prob), ("trace_path", trace_path)):
            object.__setattr__(self, name, val)
        if kind not in KINDS:
            raise ConfigurationError(f"unknown workload kind {kind!r}")
        if kind == "trace":
            if not trace_path:
                raise ConfigurationError("trace workloads need trace_path")
            return
        if distinct_items < 1:
            raise ConfigurationError("distinct_items must be >= 1")
        if total_ops < 0:
            raise ConfigurationError("total_ops must be >= 0")
        if kind == "zipf" and not zipf_skew > 0:
            raise ConfigurationError("zipf_skew must be > 0")
        if deletion_mode not in DELETION_MODES:
            raise ConfigurationError(f"unknown deletion mode {deletion_mode!r}")
        if deletion_mode == "interleaved" and not 0.0 <= delete_prob < 1.0:
            raise ConfigurationError("interleaved delete_prob must lie in [0, 1)")

    def __setattr__(self, name, value):
        raise AttributeError("WorkloadSpec is immutable")


class Workload:
    """A materialised stream: ``ops`` (uint8), ``keys`` (uint64) and, for
    synthetic streams, ``ranks`` (int64), as CUDA tensors."""

    def __init__(self, spec, ops, keys, ranks=None):
        self.spec = spec
        self.ops = ops
        self.keys = keys
        self.ranks = ranks

    def __len__(self):
        return int(self.ops.shape[0])

    def operations(self):
        for op, key in zip(self.ops.cpu().numpy(), self.keys.cpu().numpy()):
            yield Operation("insert" if op == 0 else "delete", int(key))


def zipf_probabilities(v: int, skew: float) -> np.ndarray:
    """P(rank r) proportional to 1/(r+1)**skew (``workloads.py:92-96``)."""
    weights = 1.0 / np.power(np.arange(1, v + 1, dtype=np.float64), skew)
    return weights / weights.sum()


def generate(spec: WorkloadSpec) -> Workload:
    """``workloads.generate`` (``workloads.py:106-131``) with the draws on the
    GPU. Zipf ranks: the numpy PCG64 stream of ``spec.seed`` evaluated in
    parallel on the device (``sfk_pcg64_draws``) and searched in the same
    float64 CDF. Uniform ranks follow numpy's bounded-integer sampler
    (Lemire with rejection): acceptance depends only on each 32-bit draw, so
    the accepted positions are flagged and compacted in parallel
    (``sfk_pcg64_bounded``). The interleaved-deletion walk runs on the device
    (one thread: every step depends on the live-item set)."""
    import torch

    from . import _lib
    from ._ops import device

    if spec.kind == "trace":
        ops, keys = load_trace(spec.trace_path)
        return Workload(spec, ops, keys)
    dev = device()
    L = _lib.lib()
    n, v = int(spec.total_ops), int(spec.distinct_items)
    rng = np.random.Generator(np.random.PCG64(spec.seed))
    st = rng.bit_generator.state["state"]
    m64 = (1 << 64) - 1
    sh, sl, ih, il = st["state"] >> 64, st["state"] & m64, st["inc"] >> 64, st["inc"] & m64

    def draws(offset, count, cdf=None):
        if cdf is not None:
            out = torch.empty(max(count, 1), dtype=torch.int64, device=dev)
            _lib.check(L.sfk_pcg64_draws(sh, sl, ih, il, offset, count, cdf.data_ptr(), cdf.numel(), out.data_ptr(),
                                         None, _lib.stream_ptr()), "sfk_pcg64_draws")
        else:
            out = torch.empty(max(count, 1), dtype=torch.float64, device=dev)
            _lib.check(L.sfk_pcg64_draws(sh, sl, ih, il, offset, count, None, 0, None, out.data_ptr(),
                                         _lib.stream_ptr()), "sfk_pcg64_draws")
        return out[:count]

    used = 0  # stream position (64-bit draws) after the candidate draws
    if spec.kind == "uniform":
        cand = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
        ws = torch.empty(int(L.sfk_pcg64_bounded_workspace_size(n, v)), dtype=torch.uint8, device=dev)
        nxt = np.zeros(1, dtype=np.int64)
        _lib.check(L.sfk_pcg64_bounded(sh, sl, ih, il, 0, n, v, cand.data_ptr(), nxt.ctypes.data, ws.data_ptr(),
                                       ws.numel(), _lib.stream_ptr()), "sfk_pcg64_bounded")
        cand = cand[:n]
        used = int(nxt[0])
    else:
        cdf = np.cumsum(zipf_probabilities(v, spec.zipf_skew))
        cdf[-1] = 1.0  # the reference's guard: every draw lands inside
        cand = draws(0, n, torch.from_numpy(cdf).to(dev))
        used = n
    if spec.deletion_mode == "none":
        ops = torch.zeros(n, dtype=torch.uint8, device=dev)
        ranks = cand
    elif spec.deletion_mode == "reverse_order":
        ops = torch.cat([torch.zeros(n, dtype=torch.uint8, device=dev), torch.ones(n, dtype=torch.uint8, device=dev)])
        ranks = torch.cat([cand, torch.flip(cand, [0])])
    else:
        decide = draws(used, n)
        pick = draws(used + n, n)
        ops = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
        ranks = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
        ws = torch.empty(int(L.sfk_interleave_workspace_size(v)), dtype=torch.uint8, device=dev)
        _lib.check(L.sfk_interleave_deletions(cand.data_ptr(), decide.data_ptr(), pick.data_ptr(),
                                              float(spec.delete_prob), n, v, ops.data_ptr(), ranks.data_ptr(),
                                              ws.data_ptr(), ws.numel(), _lib.stream_ptr()), "sfk_interleave_deletions")
        ops, ranks = ops[:n], ranks[:n]
    keys = torch.empty(ranks.numel(), dtype=torch.uint64, device=dev)
    if ranks.numel():
        _lib.check(L.sfk_mix_batch(ranks.data_ptr(), ranks.numel(), keys.data_ptr(), _lib.stream_ptr()),
                   "sfk_mix_batch")
    return Workload(spec, ops, keys, ranks)
