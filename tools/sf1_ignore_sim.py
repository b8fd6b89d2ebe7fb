"""SF1 what-if: run-collapsed dependency depth of a cfg-4
style stream with and without dropping ignorable (op, row) pairs. Insert-only
slim cells never drop below the net count of any key that maps to them. So an
insert whose own fat count in row i is at most the net count of the cell's
previous op's key can neither read nor raise that cell. Host-only (numba).
Usage: python tools/sf1_ignore_sim.py [n_ops]"""
import sys, numpy as np
sys.path.insert(0, '/root/repo')
from numba import njit
from paper_1701_04148_b200 import workloads as W
from paper_1701_04148_b200.hashing import seed_array
from oracle import oracle as orc

@njit(cache=True)
def mix(x):
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))

@njit(cache=True)
def sim(keys, kid, sseeds, fseeds, w, wp, use_ign):
    n = keys.shape[0]; d = sseeds.shape[0]
    fat = np.zeros((d, wp), np.int64)
    last_op = np.full(d * w, -1, np.int64); last_any = np.full(d * w, -1, np.int64)
    level = np.zeros(n, np.int64)
    Nk = np.zeros(n, np.int64); cnt = np.zeros(kid.max() + 1, np.int64)
    cells = np.empty(d, np.int64); ign = np.zeros(d, np.bool_)
    maxlev = 0; nruns = 0; nign = 0
    for t in range(n):
        k = np.uint64(keys[t])
        for i in range(d):
            cells[i] = i * w + np.int64(mix(k ^ sseeds[i]) % np.uint64(w))
            f = np.int64(mix(k ^ fseeds[i]) % np.uint64(wp))
            fat[i, f] += 1
            oa = fat[i, f]
            p = last_any[cells[i]]
            ign[i] = use_ign and p >= 0 and Nk[p] >= oa
            if ign[i]: nign += 1
        cnt[kid[t]] += 1
        Nk[t] = cnt[kid[t]]
        pf = -1; cont = True; anyc = False
        for i in range(d):
            if ign[i]: continue
            anyc = True
            q = last_op[cells[i]]
            if q < 0: cont = False; continue
            if pf == -1: pf = q
            elif pf != q: cont = False
        if cont and anyc and pf >= 0 and keys[pf] == keys[t]:
            level[t] = level[pf]
        else:
            nruns += 1
            lev = 0
            for i in range(d):
                if ign[i]: continue
                q = last_op[cells[i]]
                if q >= 0 and level[q] + 1 > lev: lev = level[q] + 1
            if lev == 0: lev = 1
            level[t] = lev
            if lev > maxlev: maxlev = lev
        for i in range(d):
            last_any[cells[i]] = t
            if not ign[i]: last_op[cells[i]] = t
    return maxlev, nruns, nign

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20_000_000
c = W.cfg4(seed=2017, n=n, v=n // 10)
keys = orc.keys_from_records(c["records"])
_, kid = np.unique(keys, return_inverse=True)
for use in (False, True):
    print("cfg4 n", n, "ignore" if use else "plain", sim(keys, kid.astype(np.int64), seed_array(2017, 0, 4), seed_array(2017, 4, 4), 12800, 4194304, use), flush=True)
