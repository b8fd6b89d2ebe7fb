"""SFF what-if: run-collapsed engine depth of the cfg-3
streams when provably ignorable (op, row) pairs leave the cells' sequences,
with VALID lower bounds (tools/sff_ignore_sim.py used the historical maximum
of key counts, which deletes invalidate, and its masks fragmented the hot
key's runs).

Facts (well-formed batch: no key's batch-local net count ever < 0, and
S[c] <= max fat slot of bucket c at batch start):
  * S[c](t) >= L_y(t) for every key y on c (L = batch-local net count);
  * an insert of x drops row i when LB(c_i) >= b_min(x): c_i is then neither
    the min nor raised, and m's comparison with b_min is unchanged;
  * a delete of x drops row i when x's slot is not the bucket's unique
    maximum (the clamp is then a no-op: S <= max fat stays).
LB choices: 'dom' = L of the cell's dominant key (most batch ops on the
cell), 'max' = max over all keys on c of their current L (exact bound).
Run rule: consecutive ops of one key whose non-dropped cells have no other
non-dropped op in between; 'eqmask' also requires equal drop masks.
Host-only (numba). Prints (levels, runs, dropped pairs)."""
import sys

import numpy as np
from numba import njit

sys.path.insert(0, "/root/repo")
from paper_1701_04148_b200 import workloads as W  # noqa: E402
from paper_1701_04148_b200.hashing import seed_array  # noqa: E402


@njit(cache=True)
def mix(x):
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


@njit(cache=True)
def cells_of(keys, bseeds, sseeds, w, z):
    n = keys.shape[0]
    d = bseeds.shape[0]
    cl = np.empty((n, d), np.int64)
    sl = np.empty((n, d), np.int64)
    for t in range(n):
        k = np.uint64(keys[t])
        for i in range(d):
            cl[t, i] = i * w + np.int64(mix(k ^ bseeds[i]) % np.uint64(w))
            sl[t, i] = np.int64(mix(k ^ sseeds[i]) % np.uint64(z))
    return cl, sl


@njit(cache=True)
def dominant(cl, kid, nk, ncell):
    # per cell: key with most ops on it (ties: smaller id); via per-key totals
    tot = np.zeros(nk, np.int64)
    for t in range(kid.shape[0]):
        tot[kid[t]] += 1
    dom = np.full(ncell, -1, np.int64)
    for t in range(kid.shape[0]):
        k = kid[t]
        for i in range(cl.shape[1]):
            c = cl[t, i]
            q = dom[c]
            if q < 0 or tot[k] > tot[q] or (tot[k] == tot[q] and k < q):
                dom[c] = k
    return dom


@njit(cache=True)
def sim(cl, sl, ops, kid, nk, w, z, lbmode, eqmask, cell_keys_ptr, cell_keys, fatrule=0):
    n, d = cl.shape
    ncell = d * w
    fat = np.zeros((ncell, z), np.int64)
    last_op = np.full(ncell, -1, np.int64)
    level = np.zeros(n, np.int64)
    cnt = np.zeros(nk, np.int64)
    lastmask = np.full(nk, -1, np.int64)
    dom = dominant(cl, kid, nk, ncell) if lbmode == 1 else np.zeros(1, np.int64)
    ign = np.zeros(d, np.bool_)
    own_a = np.zeros((n, d), np.int64)
    oth_a = np.zeros((n, d), np.int64)
    kprev = np.full(nk, -1, np.int64)
    maxlev = 0
    nruns = 0
    nign = 0
    for t in range(n):
        x = kid[t]
        op = ops[t]
        bmin = 1 << 62
        for i in range(d):
            c = cl[t, i]
            s = sl[t, i]
            ob = fat[c, s]
            fat[c, s] += 1 if op == 0 else -1
            oa = fat[c, s]
            if oa < bmin:
                bmin = oa
            om = 0
            for q in range(z):
                if q != s and fat[c, q] > om:
                    om = fat[c, q]
            ign[i] = (ob <= om) if (op == 1 and lbmode > 0) else False
            own_a[t, i] = oa
            oth_a[t, i] = om
        if op == 0 and lbmode > 0:
            for i in range(d):
                c = cl[t, i]
                lb = -1
                if lbmode == 1:
                    y = dom[c]
                    if y != x:
                        lb = cnt[y]
                else:
                    for p in range(cell_keys_ptr[c], cell_keys_ptr[c + 1]):
                        y = cell_keys[p]
                        if y != x and cnt[y] > lb:
                            lb = cnt[y]
                if lb >= bmin:
                    ign[i] = True
        cnt[x] += 1 if op == 0 else -1
        mask = 0
        for i in range(d):
            if ign[i]:
                mask |= 1 << i
                nign += 1
        pf = -1
        cont = True
        anyc = False
        for i in range(d):
            if ign[i]:
                continue
            anyc = True
            q = last_op[cl[t, i]]
            if q < 0:
                cont = False
                continue
            if pf == -1:
                pf = q
            elif pf != q:
                cont = False
        if fatrule > 0 and cont and anyc and pf >= 0 and kid[pf] == x:
            # the closed forms track the key's own slot counts from the head and
            # use the head's max-of-other-slots: a dropped foreign op that
            # changed either breaks the run (fatrule 1); fatrule 2 keeps it when
            # the other slots cannot bind at either op (caps = own counts)
            dl = 1 if op == 0 else -1
            for i in range(d):
                if own_a[t, i] != own_a[pf, i] + dl:
                    cont = False
                if oth_a[t, i] != oth_a[pf, i]:
                    if fatrule == 1:
                        cont = False
                    else:
                        bind_t = op == 1 and oth_a[t, i] > own_a[t, i]
                        bind_p = ops[pf] == 1 and oth_a[pf, i] > own_a[pf, i]
                        if bind_t or bind_p:
                            cont = False
        if cont and anyc and pf >= 0 and kid[pf] == x and (not eqmask or lastmask[x] == mask):
            level[t] = level[pf]
        else:
            nruns += 1
            lev = 0
            for i in range(d):
                if ign[i]:
                    continue
                q = last_op[cl[t, i]]
                if q >= 0 and level[q] + 1 > lev:
                    lev = level[q] + 1
            if lev == 0:
                lev = 1
            level[t] = lev
            if lev > maxlev:
                maxlev = lev
        lastmask[x] = mask
        for i in range(d):
            if not ign[i]:
                last_op[cl[t, i]] = t
    return maxlev, nruns, nign


def cell_key_lists(cl, kid, ncell):
    c = cl.reshape(-1)
    k = np.repeat(kid, cl.shape[1])
    pairs = np.unique(c * (kid.max() + 1) + k)
    cc = pairs // (kid.max() + 1)
    kk = pairs % (kid.max() + 1)
    ptr = np.zeros(ncell + 1, np.int64)
    np.add.at(ptr, cc + 1, 1)
    return np.cumsum(ptr), kk.astype(np.int64)


if __name__ == "__main__":
    alphas = [float(a) for a in sys.argv[1].split(",")] if len(sys.argv) > 1 else [1.0, 0.5, 1.5]
    for a in alphas:
        c = W.cfg3(seed=2017, alpha=a)
        keys = c["keys"].astype(np.uint64)
        ops = c["ops"]
        _, kid = np.unique(keys, return_inverse=True)
        kid = kid.astype(np.int64)
        nk = int(kid.max()) + 1
        cl, sl = cells_of(keys, seed_array(2017, 0, 4), seed_array(2017, 4, 4), 65536, 4)
        ptr, ck = cell_key_lists(cl, kid, 4 * 65536)
        for lbmode, eqm, fr in ((0, True, 0), (1, True, 0), (1, True, 1), (1, True, 2), (2, True, 1)):
            r = sim(cl, sl, ops, kid, nk, 65536, 4, lbmode, eqm, ptr, ck, fr)
            print("alpha", a, "lb", ["none", "dom", "max"][lbmode], "eqmask" if eqm else "anymask",
                  ["fat-ignored", "fat-strict", "fat-relaxed"][fr], r, flush=True)
