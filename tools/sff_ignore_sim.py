"""SFF what-if: run-collapsed depth of the cfg-3 streams
when ignorable (op, row) pairs leave the cells' sequences. An insert
ignores a row whose cell's running max of key net counts reaches its b_min
(valid for well-formed batches). A delete ignores a row whose slot is not
the bucket's unique max. Runs need equal drop masks. Host-only (numba)."""
import sys, numpy as np
sys.path.insert(0, '/root/repo')
from numba import njit
from paper_1701_04148_b200 import workloads as W
from paper_1701_04148_b200.hashing import seed_array

@njit(cache=True)
def mix(x):
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))

@njit(cache=True)
def sim(keys, ops, kid, bseeds, sseeds, w, z, mode, row0):
    # mode 0 plain, 1 ignore with per-cell prefix max of key net counts (reset never; valid for well-formed streams)
    n = keys.shape[0]; d = bseeds.shape[0]
    fat = np.zeros((d, w, z), np.int64)
    last_op = np.full(d * w, -1, np.int64); pmax = np.zeros(d * w, np.int64)
    level = np.zeros(n, np.int64); cnt = np.zeros(kid.max() + 1, np.int64)
    cells = np.empty(d, np.int64); slots = np.empty(d, np.int64); ign = np.zeros(d, np.bool_)
    maxlev = 0; nruns = 0; nign = 0
    lastmask = np.zeros(kid.max() + 1, np.int64)
    for t in range(n):
        k = np.uint64(keys[t]); op = ops[t]
        own_after = np.empty(d, np.int64)
        bmin = 1 << 62
        mask = 0
        for i in range(d):
            cells[i] = i * w + np.int64(mix(k ^ bseeds[i]) % np.uint64(w))
            slots[i] = np.int64(mix(k ^ sseeds[i]) % np.uint64(z))
            j = cells[i] - i * w
            ob = fat[i, j, slots[i]]
            fat[i, j, slots[i]] += 1 if op == 0 else -1
            oa = fat[i, j, slots[i]]; own_after[i] = oa
            if oa < bmin: bmin = oa
            om = 0
            for s in range(z):
                if s != slots[i] and fat[i, j, s] > om: om = fat[i, j, s]
            ig = False
            if mode == 1 and (i > 0 or not row0):
                if op == 1: ig = ob <= om
            ign[i] = ig
        if mode == 1 and op == 0:
            for i in range(d):
                if (i > 0 or not row0) and pmax[cells[i]] >= bmin: ign[i] = True
        for i in range(d):
            if ign[i]: mask |= 1 << i; nign += 1
        cnt[kid[t]] += 1 if op == 0 else -1
        pf = -1; cont = True; anyc = False
        for i in range(d):
            if ign[i]: continue
            anyc = True
            q = last_op[cells[i]]
            if q < 0: cont = False; continue
            if pf == -1: pf = q
            elif pf != q: cont = False
        if cont and anyc and pf >= 0 and keys[pf] == keys[t] and lastmask[kid[t]] == mask:
            level[t] = level[pf]
        else:
            nruns += 1; lev = 0
            for i in range(d):
                if ign[i]: continue
                q = last_op[cells[i]]
                if q >= 0 and level[q] + 1 > lev: lev = level[q] + 1
            if lev == 0: lev = 1
            level[t] = lev
            if lev > maxlev: maxlev = lev
        lastmask[kid[t]] = mask
        for i in range(d):
            if cnt[kid[t]] > pmax[cells[i]]: pmax[cells[i]] = cnt[kid[t]]
            if not ign[i]: last_op[cells[i]] = t
    return maxlev, nruns, nign

for a in (1.0, 0.5):
    c = W.cfg3(seed=2017, alpha=a)
    keys = c["keys"].astype(np.uint64); ops = c["ops"]
    _, kid = np.unique(keys, return_inverse=True)
    bs = seed_array(2017, 0, 4); ss = seed_array(2017, 4, 4)
    for mode, row0 in ((0, True), (1, True), (1, False)):
        print("alpha", a, "mode", mode, "row0-kept" if row0 else "all-rows", sim(keys, ops, kid.astype(np.int64), bs, ss, 65536, 4, mode, row0), flush=True)
