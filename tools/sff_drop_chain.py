"""Critical chain of the cfg-3 engine under tools/sff_drop_sim2.py's valid drop rules
(dominant-key lower bound, delete no-op rule), classifying why each run on the
chain starts: first op of its key, a kept foreign op on a kept cell, a drop-mask
change, a foreign op that moved the key's own slot count (own), or one that moved
the max of the other slots (others). Usage: python tools/sff_drop_chain.py ALPHA FATRULE
(FATRULE 0 ignores the closed forms' fat inputs, 1 breaks on any change, 2 only
when the other slots can bind). Host-only (numba)."""
import sys, numpy as np
sys.path.insert(0, '/root/repo/tools'); sys.path.insert(0, '/root/repo')
from numba import njit
from collections import Counter
from sff_drop_sim2 import cells_of, dominant
from paper_1701_04148_b200 import workloads as W
from paper_1701_04148_b200.hashing import seed_array

@njit(cache=True)
def sim(cl, sl, ops, kid, nk, w, z, fatrule):
    n, d = cl.shape
    ncell = d * w
    fat = np.zeros((ncell, z), np.int64)
    last_op = np.full(ncell, -1, np.int64)
    level = np.zeros(n, np.int64); parent = np.full(n, -1, np.int64); head = np.full(n, -1, np.int64)
    why = np.zeros(n, np.int64)
    cnt = np.zeros(nk, np.int64)
    lastmask = np.full(nk, -1, np.int64)
    dom = dominant(cl, kid, nk, ncell)
    ign = np.zeros(d, np.bool_)
    own_a = np.zeros((n, d), np.int64); oth_a = np.zeros((n, d), np.int64)
    kprev = np.full(nk, -1, np.int64)
    for t in range(n):
        x = kid[t]; op = ops[t]; bmin = 1 << 62
        for i in range(d):
            c = cl[t, i]; s = sl[t, i]
            ob = fat[c, s]; fat[c, s] += 1 if op == 0 else -1; oa = fat[c, s]
            if oa < bmin: bmin = oa
            om = 0
            for q in range(z):
                if q != s and fat[c, q] > om: om = fat[c, q]
            ign[i] = (ob <= om) if op == 1 else False
            own_a[t, i] = oa; oth_a[t, i] = om
        if op == 0:
            for i in range(d):
                y = dom[cl[t, i]]
                if y != x and cnt[y] >= bmin: ign[i] = True
        cnt[x] += 1 if op == 0 else -1
        mask = 0
        for i in range(d):
            if ign[i]: mask |= 1 << i
        kp = kprev[x]
        # why the run would break, in priority order
        reason = 0
        if kp < 0: reason = 1  # first op of key
        else:
            for i in range(d):
                if ign[i]: continue
                if last_op[cl[t, i]] != kp: reason = 2  # a kept foreign op on a kept cell (or cell newly kept)
            if reason == 0 and lastmask[x] != mask: reason = 3
            if reason == 0 and fatrule > 0:
                dl = 1 if op == 0 else -1
                for i in range(d):
                    if own_a[t, i] != own_a[kp, i] + dl: reason = 4
                if reason == 0:
                    for i in range(d):
                        if oth_a[t, i] != oth_a[kp, i]:
                            if fatrule == 1: reason = 5
                            else:
                                if (op == 1 and oth_a[t, i] > own_a[t, i]) or (ops[kp] == 1 and oth_a[kp, i] > own_a[kp, i]): reason = 5
            if mask == (1 << d) - 1: reason = 6
        if reason == 0:
            level[t] = level[kp]; parent[t] = parent[kp]; head[t] = head[kp]
        else:
            lev = 0; par = -1
            for i in range(d):
                if ign[i]: continue
                q = last_op[cl[t, i]]
                if q >= 0 and level[q] + 1 > lev: lev = level[q] + 1; par = q
            if lev == 0: lev = 1
            level[t] = lev; parent[t] = par; head[t] = t; why[t] = reason
        lastmask[x] = mask; kprev[x] = t
        for i in range(d):
            if not ign[i]: last_op[cl[t, i]] = t
    return level, parent, head, why

a = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
fr = int(sys.argv[2]) if len(sys.argv) > 2 else 1
c = W.cfg3(seed=2017, alpha=a)
keys = c["keys"].astype(np.uint64); ops = c["ops"]
uniq, kid, cnts = np.unique(keys, return_inverse=True, return_counts=True)
kid = kid.astype(np.int64)
order = np.argsort(-cnts); rankof = np.empty_like(order); rankof[order] = np.arange(order.size)
cl, sl = cells_of(keys, seed_array(2017, 0, 4), seed_array(2017, 4, 4), 65536, 4)
level, parent, head, why = sim(cl, sl, ops, kid, int(kid.max()) + 1, 65536, 4, fr)
t = int(np.argmax(level)); chain = []
while t >= 0:
    chain.append(t); p = parent[head[t]]; t = int(p) if p >= 0 else -1
print("levels", level.max(), "chain", len(chain), "runs", int((head == np.arange(len(head))).sum()))
wh = Counter(int(why[head[t]]) for t in chain)
rk = Counter(min(int(rankof[kid[t]]) // 100, 20) for t in chain)
ks = Counter(int(rankof[kid[t]]) for t in chain)
print("why (1 first,2 kept-foreign,3 mask,4 own,5 others,6 all-dropped):", sorted(wh.items()))
print("rank buckets x100:", sorted(rk.items())); print("top ranks on chain:", ks.most_common(8))
print("ops on chain:", Counter(int(ops[t]) for t in chain))
