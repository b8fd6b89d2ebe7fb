"""What-if for the ordered engine: the run-collapsed
dependency depth of the cfg-3 streams if runs could merge across keys
(union of the runs an op depends on, capped at `cap` slim cells), replayed
sequentially by one lane. Host-only (numba); prints (levels, runs) per cap.
cap = 4 reproduces the engine's current run definition and its measured
critical-path hop counts (1794 / 6498 / 3012 at alpha = 0.5 / 1.0 / 1.5)."""
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
def find(par, x):
    while par[x] != x:
        par[x] = par[par[x]]; x = par[x]
    return x

@njit(cache=True)
def sim(keys, bseeds, w, cap):
    n = keys.shape[0]; d = bseeds.shape[0]
    last_run = np.full(d * w, -1, np.int64)
    par = np.arange(n); lev = np.zeros(n, np.int64); ncell = np.zeros(n, np.int64); nops = np.zeros(n, np.int64)
    cells = np.empty(d, np.int64); roots = np.empty(d, np.int64)
    nr = 0; maxlev = 0
    for t in range(n):
        k = np.uint64(keys[t])
        for i in range(d):
            cells[i] = i * w + np.int64(mix(k ^ bseeds[i]) % np.uint64(w))
        nroots = 0; tot = 0; newcells = 0
        for i in range(d):
            q = last_run[cells[i]]
            if q < 0:
                newcells += 1; continue
            r = find(par, q)
            dup = False
            for z in range(nroots):
                if roots[z] == r: dup = True
            if not dup:
                roots[nroots] = r; nroots += 1; tot += ncell[r]
        if nroots >= 1 and tot + newcells <= cap:
            # merge all roots, add t
            r0 = roots[0]; L = lev[r0]
            for z in range(1, nroots):
                r = roots[z]; par[r] = r0; ncell[r0] += ncell[r]; nops[r0] += nops[r]
                if lev[r] > L: L = lev[r]
            lev[r0] = L; ncell[r0] += newcells; nops[r0] += 1
            R = r0
        else:
            R = t; nr += 1
            L = 0
            for z in range(nroots):
                if lev[roots[z]] + 1 > L: L = lev[roots[z]] + 1
            if L == 0: L = 1
            lev[R] = L; ncell[R] = d; nops[R] = 1
        if lev[R] > maxlev: maxlev = lev[R]
        for i in range(d):
            last_run[cells[i]] = R
    return maxlev, nr

for a in (0.5, 1.0, 1.5):
    c = W.cfg3(seed=2017, alpha=a)
    keys = c["keys"].astype(np.uint64)
    for cap in (4, 7, 8, 12, 16):
        print("alpha", a, "cap", cap, sim(keys, seed_array(2017, 0, 4), 65536, cap), flush=True)
