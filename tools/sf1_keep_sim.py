"""SF1 what-if for the cfg-4 pipeline (DESIGN.md §3.2a, §8 item 3): how many
(op, row) pairs survive the drop rule under different lower bounds of a slim
cell. Every bound is valid (an SF1 cell is >= the batch count of every key
seen on it earlier); they differ in what they cost on the GPU.

  tile   today's rule: running max of the key counts of earlier ops on the
         cell inside the same 2048-element tile of the cell-sorted pairs
  chunk  op-order rule: max key count of the cell's ops in earlier stream
         chunks of C ops (per-chunk shared-memory tables, prefix max over
         chunks); no cell-order gather
  exact  the previous op on the cell (upper limit of any bound of this kind)

The drop test is lb >= b_min(t) (exact per-op b_min). Host-only (numba).
Usage: python tools/sf1_keep_sim.py [n_ops] [chunk_ops]"""
import sys

import numpy as np
from numba import njit

sys.path.insert(0, "/root/repo")
from oracle import oracle as orc  # noqa: E402
from paper_1701_04148_b200 import workloads as W  # noqa: E402
from paper_1701_04148_b200.hashing import seed_array  # noqa: E402


@njit(cache=True)
def mix(x):
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


@njit(cache=True)
def prep(keys, kid, sseeds, fseeds, w, wp):
    n = keys.shape[0]
    d = sseeds.shape[0]
    fat = np.zeros((d, wp), np.int64)
    cells = np.empty((n, d), np.int32)
    bmin = np.empty(n, np.int64)
    cnt = np.zeros(kid.max() + 1, np.int64)
    kc = np.empty(n, np.int64)
    for t in range(n):
        k = np.uint64(keys[t])
        b = np.int64(1) << 62
        for i in range(d):
            cells[t, i] = i * w + np.int64(mix(k ^ sseeds[i]) % np.uint64(w))
            f = np.int64(mix(k ^ fseeds[i]) % np.uint64(wp))
            fat[i, f] += 1
            if fat[i, f] < b:
                b = fat[i, f]
        bmin[t] = b
        cnt[kid[t]] += 1
        kc[t] = cnt[kid[t]]
    return cells, bmin, kc


@njit(cache=True)
def keep_exact(cells, bmin, kc):
    n, d = cells.shape
    last = np.full(d * 65536 * 4, -1, np.int64)
    kept = 0
    kops = 0
    for t in range(n):
        any_k = False
        for i in range(d):
            c = cells[t, i]
            p = last[c]
            if not (p >= 0 and kc[p] >= bmin[t]):
                kept += 1
                any_k = True
            last[c] = t
        if any_k:
            kops += 1
    return kept, kops


@njit(cache=True)
def keep_chunk(cells, bmin, kc, C, ncells):
    n, d = cells.shape
    carry = np.zeros(ncells, np.int64)
    cur = np.zeros(ncells, np.int64)
    kept = 0
    kops = 0
    for t0 in range(0, n, C):
        t1 = min(n, t0 + C)
        for t in range(t0, t1):
            any_k = False
            for i in range(d):
                if not (carry[cells[t, i]] >= bmin[t]):
                    kept += 1
                    any_k = True
            if any_k:
                kops += 1
        for t in range(t0, t1):
            for i in range(d):
                c = cells[t, i]
                if kc[t] > cur[c]:
                    cur[c] = kc[t]
        for c in range(ncells):
            carry[c] = cur[c]
    return kept, kops


def keep_tile(cells, bmin, kc, tile=2048):
    n, d = cells.shape
    flat_c = cells.T.reshape(-1).astype(np.int64)  # row-major pairs (row i block = op order)
    flat_t = np.tile(np.arange(n, dtype=np.int64), d)
    order = np.lexsort((flat_t, flat_c))
    sc = flat_c[order]
    st = flat_t[order]
    return _tile(sc, st, bmin, kc, tile)


@njit(cache=True)
def _tile(sc, st, bmin, kc, tile):
    N = sc.shape[0]
    kept = 0
    keptop = np.zeros(bmin.shape[0], np.uint8)
    run = 0
    for e in range(N):
        head = e == 0 or sc[e - 1] != sc[e]
        if e % tile == 0 or head:
            lb = 0
            hasprev = False
        else:
            lb = run
            hasprev = True
        t = st[e]
        if not (hasprev and lb >= bmin[t]):
            kept += 1
            keptop[t] = 1
        if e % tile == 0 or head:
            run = kc[t]
        else:
            run = max(run, kc[t])
    return kept, int(keptop.sum())


n = int(sys.argv[1]) if len(sys.argv) > 1 else 20_000_000
C = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
c = W.cfg4(seed=2017, n=n, v=max(n // 10, 1))
keys = orc.keys_from_records(c["records"])
del c
_, kid = np.unique(keys, return_inverse=True)
cells, bmin, kc = prep(keys, kid.astype(np.int64), seed_array(2017, 0, 4), seed_array(2017, 4, 4), 12800, 4194304)
N = 4 * n
print(f"n={n} pairs={N}")
k, o = keep_exact(cells, bmin, kc)
print(f"exact prev op : kept pairs {k} ({k / N:.3f}), ops with a kept row {o} ({o / n:.3f})", flush=True)
k, o = keep_tile(cells, bmin, kc)
print(f"tile 2048     : kept pairs {k} ({k / N:.3f}), ops with a kept row {o} ({o / n:.3f})", flush=True)
for CC in ((C,) if len(sys.argv) > 3 else (C // 4, C, C * 4)):
    k, o = keep_chunk(cells, bmin, kc, CC, 4 * 12800)
    print(f"chunk {CC:7d} : kept pairs {k} ({k / N:.3f}), ops with a kept row {o} ({o / n:.3f})", flush=True)


# ---------------------------------------------------------------- engine depth
@njit(cache=True)
def depth(cells, kid, drop):
    """Critical-path levels and runs of the run-collapsed engine for the given
    (op, row) drop flags: a run continues from the key's previous op when
    every kept row's previous kept op is that op and the drop masks agree."""
    n, d = cells.shape
    last = np.full(d * 65536 * 4, -1, np.int64)
    kprev_op = np.full(kid.max() + 1, -1, np.int64)
    level = np.zeros(n, np.int64)
    mask = np.zeros(n, np.int64)
    maxlev = 0
    runs = 0
    for t in range(n):
        m = 0
        for i in range(d):
            if drop[t, i]:
                m |= 1 << i
        mask[t] = m
        p = kprev_op[kid[t]]
        kprev_op[kid[t]] = t
        if m == (1 << d) - 1:
            level[t] = 0
            continue
        cont = p >= 0 and mask[p] == m
        if cont:
            for i in range(d):
                if not drop[t, i] and last[cells[t, i]] != p:
                    cont = False
        if cont:
            level[t] = level[p]
        else:
            runs += 1
            lev = 1
            for i in range(d):
                if not drop[t, i]:
                    q = last[cells[t, i]]
                    if q >= 0 and level[q] + 1 > lev:
                        lev = level[q] + 1
            level[t] = lev
            if lev > maxlev:
                maxlev = lev
        for i in range(d):
            if not drop[t, i]:
                last[cells[t, i]] = t
    return maxlev, runs


@njit(cache=True)
def drop_chunk(cells, bmin, kc, C, ncells):
    n, d = cells.shape
    drop = np.zeros((n, d), np.bool_)
    carry = np.zeros(ncells, np.int64)
    for t0 in range(0, n, C):
        t1 = min(n, t0 + C)
        for t in range(t0, t1):
            for i in range(d):
                drop[t, i] = carry[cells[t, i]] >= bmin[t]
        for t in range(t0, t1):
            for i in range(d):
                c = cells[t, i]
                if kc[t] > carry[c]:
                    carry[c] = kc[t]
    return drop


@njit(cache=True)
def _tile_drop(sc, st, srow, bmin, kc, tile, drop):
    N = sc.shape[0]
    run = 0
    for e in range(N):
        head = e == 0 or sc[e - 1] != sc[e]
        t = st[e]
        if not (e % tile == 0 or head) and run >= bmin[t]:
            drop[t, srow[e]] = True
        if e % tile == 0 or head:
            run = kc[t]
        else:
            run = max(run, kc[t])


def drop_tile(cells, bmin, kc, tile=2048):
    n, d = cells.shape
    flat_c = cells.T.reshape(-1).astype(np.int64)
    flat_t = np.tile(np.arange(n, dtype=np.int64), d)
    order = np.lexsort((flat_t, flat_c))
    drop = np.zeros((n, d), np.bool_)
    _tile_drop(flat_c[order], flat_t[order], (flat_c[order] // 12800).astype(np.int64), bmin, kc, tile, drop)
    return drop


if len(sys.argv) > 3 and sys.argv[3] == "depth":
    k64 = kid.astype(np.int64)
    print("none   ", depth(cells, k64, np.zeros(cells.shape, np.bool_)), flush=True)
    print("tile   ", depth(cells, k64, drop_tile(cells, bmin, kc)), flush=True)
    for CC in (C // 16, C // 4, C):
        print(f"chunk {CC}", depth(cells, k64, drop_chunk(cells, bmin, kc, CC, 4 * 12800)), flush=True)
