"""What-if for the ordered engine: chaining. Runs as the engine forms them
(same key, all d cells last touched by the run's previous op). A run whose
predecessor runs, after one level of transitive reduction (drop a pred that
is itself a pred of another pred), reduce to ONE run r is "direct" on r; each
run r chains at most one direct successor (the earliest), which r's lane
executes right after r with no readiness detection. Prints the critical path
in microseconds for a cost model (hop = detection + replay, chained edge =
replay only) and the hop count, with and without chaining. Host-only (numba).
Usage: python tools/chain_sim.py [alpha] [hop_us] [chain_us]"""
import sys
import numpy as np

sys.path.insert(0, '/root/repo')
from numba import njit  # noqa: E402

from paper_1701_04148_b200 import workloads as W  # noqa: E402
from paper_1701_04148_b200.hashing import seed_array  # noqa: E402


@njit(cache=True)
def mix(x):
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


@njit(cache=True)
def build_runs(keys, bseeds, w):
    n = keys.shape[0]
    d = bseeds.shape[0]
    last_op = np.full(d * w, -1, np.int64)
    run_of = np.empty(n, np.int64)
    heads = np.empty(n, np.int64)
    preds = np.full((n, d), -1, np.int64)  # per run: pred runs (by run id), -1 none
    nr = 0
    cells = np.empty(d, np.int64)
    for t in range(n):
        k = np.uint64(keys[t])
        for i in range(d):
            cells[i] = i * w + np.int64(mix(k ^ bseeds[i]) % np.uint64(w))
        p = last_op[cells[0]]
        cont = p >= 0
        for i in range(1, d):
            if last_op[cells[i]] != p:
                cont = False
        if cont and keys[p] == keys[t]:
            run_of[t] = run_of[p]
        else:
            r = nr
            nr += 1
            heads[r] = t
            run_of[t] = r
            for i in range(d):
                q = last_op[cells[i]]
                preds[r, i] = run_of[q] if q >= 0 else -1
        for i in range(d):
            last_op[cells[i]] = t
    return nr, run_of, heads[:nr], preds[:nr]


@njit(cache=True)
def is_anc(preds, q, p, depth):
    """p is a pred of q within `depth` levels."""
    d = preds.shape[1]
    for m in range(d):
        x = preds[q, m]
        if x < 0:
            continue
        if x == p:
            return True
        if depth > 1 and x > p and is_anc(preds, x, p, depth - 1):
            return True
    return False


@njit(cache=True)
def crit(nr, preds, hop, chain_c, use_chain, depth=1, pick=0):
    d = preds.shape[1]
    # effective preds after one level of transitive reduction
    direct = np.full(nr, -1, np.int64)  # the single effective pred, if any
    for r in range(nr):
        eff = -1
        neff = 0
        for i in range(d):
            p = preds[r, i]
            if p < 0:
                continue
            dup = False
            for j in range(i):
                if preds[r, j] == p:
                    dup = True
            if dup:
                continue
            red = False
            for j in range(d):
                q = preds[r, j]
                if q < 0 or q == p:
                    continue
                if is_anc(preds, q, p, depth):
                    red = True
            if red:
                continue
            if neff == 0 or eff != p:
                neff += 1
                eff = p
        if neff == 1:
            direct[r] = eff
    chained = np.zeros(nr, np.bool_)
    taken = np.zeros(nr, np.bool_)  # r already chains a successor
    if use_chain and pick == 0:
        for r in range(nr):  # earliest direct successor per pred
            p = direct[r]
            if p >= 0 and not taken[p]:
                taken[p] = True
                chained[r] = True
    if use_chain and pick == 1:
        for r in range(nr - 1, -1, -1):  # latest direct successor per pred
            p = direct[r]
            if p >= 0 and not taken[p]:
                taken[p] = True
                chained[r] = True
    fin = np.zeros(nr, np.float64)
    hops = np.zeros(nr, np.int64)
    best = 0.0
    besth = 0
    nch = 0
    for r in range(nr):
        if chained[r]:
            p = direct[r]
            fin[r] = fin[p] + chain_c
            hops[r] = hops[p]
            nch += 1
        else:
            s = 0.0
            h = 0
            for i in range(d):
                p = preds[r, i]
                if p >= 0 and fin[p] > s:
                    s = fin[p]
                    h = hops[p]
            fin[r] = s + hop
            hops[r] = h + 1
        if fin[r] > best:
            best = fin[r]
            besth = hops[r]
    ndirect = 0
    for r in range(nr):
        if direct[r] >= 0:
            ndirect += 1
    return best, besth, nch, ndirect


alpha = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
hop = float(sys.argv[2]) if len(sys.argv) > 2 else 1.2
chain_c = float(sys.argv[3]) if len(sys.argv) > 3 else 0.3
c = W.cfg3(seed=2017, alpha=alpha)
nr, run_of, heads, preds = build_runs(c["keys"].astype(np.uint64), seed_array(2017, 0, 4), 65536)
print("alpha", alpha, "runs", nr)
for use, depth, pick in ((False, 1, 0), (True, 1, 0), (True, 2, 0), (True, 3, 0), (True, 1, 1)):
    best, besth, nch, nd = crit(nr, preds, hop, chain_c, use, depth, pick)
    print(f"chaining={use} depth={depth} pick={'earliest' if pick == 0 else 'latest'}: critical {best / 1e3:.3f} ms, "
          f"non-chained hops {besth}, chained runs {nch}, direct runs {nd}", flush=True)
