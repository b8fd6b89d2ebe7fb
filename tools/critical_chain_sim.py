"""Critical chain of the ordered engine at cfg 3 (alpha = 1.0), with the
"ignorable (op, row)" rule applied: an insert ignores row i when the cell's
previous op's key already has a net count >= the op's own slot count there
(the cell then holds at least that much, so it is neither the min nor
raised); an SFF delete ignores row i when its own slot is not the bucket's
unique maximum (the clamp is then a no-op). Prints the chain length, the key
ranks on it and why its runs break. Host-only (numba)."""
import sys, numpy as np
sys.path.insert(0, '/root/repo')
from numba import njit
from paper_1701_04148_b200 import workloads as W
from paper_1701_04148_b200.hashing import seed_array
from collections import Counter

@njit(cache=True)
def mix(x):
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))

@njit(cache=True)
def sim(keys, ops, kid, bseeds, sseeds, w, z):
    n = keys.shape[0]; d = bseeds.shape[0]
    fat = np.zeros((d, w, z), np.int64)
    last_op = np.full(d * w, -1, np.int64); last_any = np.full(d * w, -1, np.int64)
    level = np.zeros(n, np.int64); parent = np.full(n, -1, np.int64); head = np.full(n, -1, np.int64)
    why = np.zeros(n, np.int64)   # for run heads: 1 = different key pred, 2 = cells differ, 3 = no pred
    Nk = np.zeros(n, np.int64); cnt = np.zeros(kid.max() + 1, np.int64)
    cells = np.empty(d, np.int64); slots = np.empty(d, np.int64); ign = np.zeros(d, np.bool_)
    for t in range(n):
        k = np.uint64(keys[t])
        for i in range(d):
            cells[i] = i * w + np.int64(mix(k ^ bseeds[i]) % np.uint64(w))
            slots[i] = np.int64(mix(k ^ sseeds[i]) % np.uint64(z))
        op = ops[t]
        for i in range(d):
            j = cells[i] - i * w
            ob = fat[i, j, slots[i]]
            fat[i, j, slots[i]] += 1 if op == 0 else -1
            oa = fat[i, j, slots[i]]
            om = 0
            for s in range(z):
                if s != slots[i] and fat[i, j, s] > om: om = fat[i, j, s]
            p = last_any[cells[i]]
            ign[i] = (p >= 0 and Nk[p] >= oa) if op == 0 else (ob <= om)
        cnt[kid[t]] += 1 if op == 0 else -1
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
            level[t] = level[pf]; parent[t] = parent[pf]; head[t] = head[pf]
        else:
            if not anyc: why[t] = 4
            elif pf < 0: why[t] = 3
            elif not cont: why[t] = 2
            else: why[t] = 1
            lev = 0; par = -1
            for i in range(d):
                if ign[i]: continue
                q = last_op[cells[i]]
                if q >= 0 and level[q] + 1 > lev: lev = level[q] + 1; par = q
            if lev == 0: lev = 1
            level[t] = lev; parent[t] = par; head[t] = t
        for i in range(d):
            last_any[cells[i]] = t
            if not ign[i]: last_op[cells[i]] = t
    return level, parent, head, why

c = W.cfg3(seed=2017, alpha=1.0)
keys = c["keys"].astype(np.uint64); ops = c["ops"]
uniq, inv, cnts = np.unique(keys, return_inverse=True, return_counts=True)
order = np.argsort(-cnts); rankof = np.empty_like(order); rankof[order] = np.arange(order.size)
level, parent, head, why = sim(keys, ops, inv.astype(np.int64), seed_array(2017, 0, 4), seed_array(2017, 4, 4), 65536, 4)
t = int(np.argmax(level)); chain = []
while t >= 0:
    chain.append(t); p = parent[head[t]]; t = int(p) if p >= 0 else -1
print("chain", len(chain))
rk = Counter(); wh = Counter(); keysc = Counter(); ops_on = Counter()
for t in chain:
    r = rankof[inv[t]]; rk[min(r // 100, 20)] += 1; wh[int(why[head[t]])] += 1; keysc[int(inv[t])] += 1; ops_on[int(ops[t])] += 1
print("rank buckets (x100):", sorted(rk.items())); print("why:", wh); print("distinct keys", len(keysc), keysc.most_common(3), "ops", ops_on)
