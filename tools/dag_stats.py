"""Run/DAG statistics of an SF stream (CPU, numba): number of runs (maximal
same-key op sequences with no foreign op on any of the key's d slim cells in
between), run-length distribution, and the critical path of the run DAG
weighted by hops (unit cost per run) and by ops (cost = run length), which
bound the ordered engine's latency."""
import os
import sys

import numpy as np
from numba import njit

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1701_04148_b200 import workloads as W  # noqa: E402
from paper_1701_04148_b200.hashing import seed_array  # noqa: E402


@njit(cache=True)
def mix(x):
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


@njit(cache=True)
def analyse(keys, seeds, w):
    n = keys.shape[0]
    d = seeds.shape[0]
    last_op = np.full(d * w, -1, np.int64)     # last op index per cell
    run_of_op = np.empty(n, np.int64)
    level_hops = np.zeros(n, np.int64)         # per run (indexed by head op)
    level_ops = np.zeros(n, np.int64)
    run_len = np.zeros(n, np.int64)
    cells = np.empty(d, np.int64)
    nruns = 0
    for t in range(n):
        k = np.uint64(keys[t])
        for i in range(d):
            cells[i] = i * w + np.int64(mix(k ^ seeds[i]) % np.uint64(w))
        p = last_op[cells[0]]
        cont = p >= 0 and keys[p] == keys[t]
        if cont:
            for i in range(1, d):
                if last_op[cells[i]] != p:
                    cont = False
        if cont:
            r = run_of_op[p]
            run_of_op[t] = r
            run_len[r] += 1
            level_ops[r] += 1
        else:
            lh = 0
            lo = 0
            for i in range(d):
                q = last_op[cells[i]]
                if q >= 0:
                    rq = run_of_op[q]
                    lh = max(lh, level_hops[rq])
                    lo = max(lo, level_ops[rq])
            run_of_op[t] = t
            run_len[t] = 1
            level_hops[t] = lh + 1
            level_ops[t] = lo + 1
            nruns += 1
        for i in range(d):
            last_op[cells[i]] = t
    return nruns, run_len, level_hops, level_ops


def main():
    alpha = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
    c = W.cfg3(seed=2017, alpha=alpha)
    keys = c["keys"].astype(np.uint64)
    seeds = seed_array(2017, 0, 4)
    nruns, run_len, lh, lo = analyse(keys, seeds, 65536)
    rl = run_len[run_len > 0]
    print(f"alpha={alpha} ops={len(keys)} runs={nruns} depth_hops={lh.max()} depth_ops={lo.max()} "
          f"maxrun={rl.max()} runs>=32={int((rl >= 32).sum())} ops_in_runs>=32={int(rl[rl >= 32].sum())} "
          f"p99run={int(np.percentile(rl, 99))}")


if __name__ == "__main__":
    main()
