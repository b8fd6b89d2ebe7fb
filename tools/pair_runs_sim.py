"""What-if for the ordered engine: critical-path TIME of the
cfg-3 build if the ops of hot keys that share a slim cell ran as one joint
run (op by op, per-op fat observations) instead of alternating single-op
runs. Time model calibrated on today's engine: a run start waits for its
cells' previous ops + H (1.2 us: detection + replay of a claimed run); ops
inside a same-key run cost RHO (closed forms); ops inside a joint run cost
RHO_J each (op-by-op replay). Groups: keys with >= T batch ops joined by
union-find over shared cells, a group capped at CAP ops. A joint run
continues while every cell of its next op was last touched by the group (or
never). Host-only (numba). Prints (critical ms, runs, joint ops)."""
import sys

import numpy as np
from numba import njit

sys.path.insert(0, "/root/repo")
sys.path.insert(0, "/root/repo/tools")
from paper_1701_04148_b200 import workloads as W  # noqa: E402
from paper_1701_04148_b200.hashing import seed_array  # noqa: E402
from sff_drop_sim2 import cells_of  # noqa: E402


@njit(cache=True)
def find(par, x):
    while par[x] != x:
        par[x] = par[par[x]]
        x = par[x]
    return x


@njit(cache=True)
def groups(cl, kid, nk, T, CAP):
    n, d = cl.shape
    tot = np.zeros(nk, np.int64)
    for t in range(n):
        tot[kid[t]] += 1
    par = np.arange(nk)
    gsum = tot.copy()
    owner = np.full(d * 65536 * 4, -1, np.int64)  # hot key seen on a cell
    for t in range(n):
        x = kid[t]
        if tot[x] < T:
            continue
        for i in range(d):
            c = cl[t, i]
            y = owner[c]
            if y < 0:
                owner[c] = x
            elif y != x:
                rx, ry = find(par, x), find(par, y)
                if rx != ry and gsum[rx] + gsum[ry] <= CAP:
                    par[ry] = rx
                    gsum[rx] += gsum[ry]
    g = np.empty(nk, np.int64)
    for k in range(nk):
        r = find(par, k)
        g[k] = r if (tot[k] >= T and gsum[r] > tot[k]) else -1 - k  # joint groups only where keys merged
    return g


@njit(cache=True)
def sim(cl, kid, g, H, RHO, RHO_J):
    n, d = cl.shape
    last = np.full(cl.max() + 1, -1, np.int64)
    fin = np.zeros(n, np.float64)
    run = np.full(n, -1, np.int64)
    nk = g.shape[0]
    glast = np.full(nk, -1, np.int64)  # joint group (root key) / own key -> its last op
    nruns = 0
    njoint = 0
    crit = 0.0
    for t in range(n):
        x = kid[t]
        gx = g[x]
        joint = gx >= 0
        slot = gx if joint else x
        q = glast[slot]
        cont = q >= 0
        # same-key rule: every cell's previous op is q (this key's previous op)
        # joint rule: every cell's previous op belongs to the group's current run (or none)
        for i in range(d):
            p = last[cl[t, i]]
            if joint:
                if p >= 0:
                    if q < 0 or g[kid[p]] != gx or run[p] != run[q]:
                        cont = False
            else:
                if p != q:
                    cont = False
        if cont:
            run[t] = run[q]
            st = fin[q]
            f = st + (RHO_J if joint else RHO)
            if joint:
                njoint += 1
        else:
            nruns += 1
            run[t] = t
            st = 0.0
            for i in range(d):
                p = last[cl[t, i]]
                if p >= 0 and fin[p] > st:
                    st = fin[p]
            f = st + H
        fin[t] = f
        if f > crit:
            crit = f
        glast[slot] = t
        for i in range(d):
            last[cl[t, i]] = t
    return crit, nruns, njoint


if __name__ == "__main__":
    a = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
    c = W.cfg3(seed=2017, alpha=a)
    keys = c["keys"].astype(np.uint64)
    _, kid = np.unique(keys, return_inverse=True)
    kid = kid.astype(np.int64)
    nk = int(kid.max()) + 1
    cl, _ = cells_of(keys, seed_array(2017, 0, 4), seed_array(2017, 4, 4), 65536, 4)
    g0 = -1 - np.arange(nk)
    base = sim(cl, kid, g0, 1.2, 0.005, 0.15)
    print("alpha", a, "today (model)", round(base[0] / 1e3, 3), "ms", base[1:], flush=True)
    for T in (300, 1000, 3000):
        for CAP in (20_000, 60_000):
            gg = groups(cl, kid, nk, T, CAP)
            for rj in (0.1, 0.2):
                r = sim(cl, kid, gg, 1.2, 0.005, rj)
                print("alpha", a, "T", T, "cap", CAP, "rho_j", rj, "->", round(r[0] / 1e3, 3), "ms", r[1:],
                      "grouped keys", int((gg >= 0).sum()), flush=True)
