"""Critical-path breakdown of the ordered slim engine from per-run GPU
timestamps (SFK_ENGINE_TRACE=1). Usage: SFK_ENGINE_TRACE=1 python tools/trace_engine.py [alpha]"""
import ctypes
import os
import sys

import numpy as np
import torch
from numba import njit

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1701_04148_b200 as P  # noqa: E402
from paper_1701_04148_b200 import _lib, workloads as W  # noqa: E402
from paper_1701_04148_b200.hashing import seed_array  # noqa: E402


@njit(cache=True)
def mix(x):
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


@njit(cache=True)
def dag(keys, seeds, w):
    n = keys.shape[0]
    d = seeds.shape[0]
    last_op = np.full(d * w, -1, np.int64)
    run_of_op = np.empty(n, np.int64)
    rid = np.full(n, -1, np.int64)      # run id by head op
    pred = np.full((n, d), -1, np.int64)
    rlen = np.zeros(n, np.int64)
    cells = np.empty(d, np.int64)
    nr = 0
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
            run_of_op[t] = run_of_op[p]
            rlen[run_of_op[p]] += 1
        else:
            r = nr
            nr += 1
            run_of_op[t] = r
            rlen[r] = 1
            for i in range(d):
                q = last_op[cells[i]]
                if q >= 0:
                    pred[r, i] = run_of_op[q]
        for i in range(d):
            last_op[cells[i]] = t
    return nr, pred[:nr], rlen[:nr]


def main():
    alpha = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
    variant = sys.argv[2] if len(sys.argv) > 2 else "sff"
    c = W.cfg3(seed=2017, alpha=alpha)
    keys = c["keys"].astype(np.uint64)
    nr, pred, rlen = dag(keys, seed_array(2017, 0, 4), 65536)
    ops_d = torch.from_numpy(c["ops"]).cuda()
    keys_d = torch.from_numpy(c["keys"]).cuda()
    for _ in range(2):
        sk = P.SfSketch(P.SketchParams(d=4, w=65536, z=4, w_prime=262144, master_seed=2017), variant)
        sk.apply_ops(ops_d, keys_d)
    torch.cuda.synchronize()
    tr = np.zeros(3 * nr, dtype=np.uint64)
    rc = _lib.load_library().sfk_engine_trace(tr.ctypes.data_as(ctypes.c_void_p), nr)
    assert rc == 0
    tr = tr.reshape(nr, 3).astype(np.int64)
    t0 = tr[:, 0].min()
    claim, ready, done = tr[:, 0] - t0, tr[:, 1] - t0, tr[:, 2] - t0
    dep_done = np.where(pred >= 0, done[np.maximum(pred, 0)], 0).max(axis=1)
    print(f"alpha={alpha} runs={nr} span={done.max() / 1e6:.2f} ms")
    # walk the critical path backwards from the last finisher
    r = int(np.argmax(done))
    hops = 0
    tot = {"replay": 0, "detect": 0, "claim_wait": 0}
    path = []
    while True:
        hops += 1
        path.append(r)
        tot["replay"] += done[r] - ready[r]
        gate = dep_done[r]
        if claim[r] > gate:  # the run was claimed after its inputs were ready
            tot["claim_wait"] += claim[r] - gate
            tot["detect"] += ready[r] - claim[r]
        else:
            tot["detect"] += ready[r] - gate
        ps = pred[r][pred[r] >= 0]
        if ps.size == 0:
            break
        r = int(ps[np.argmax(done[ps])])
    print(f"critical path: {hops} hops; replay {tot['replay'] / 1e6:.2f} ms, dependency detect "
          f"{tot['detect'] / 1e6:.2f} ms ({tot['detect'] / max(hops, 1):.0f} ns/hop), claim wait "
          f"{tot['claim_wait'] / 1e6:.2f} ms")
    path = np.array(path)
    pl = rlen[path]
    prep = (done - ready)[path]
    for lo, hi in ((1, 2), (2, 8), (8, 32), (32, 256), (256, 1024), (1024, 1 << 40)):
        sel = (pl >= lo) & (pl < hi)
        if sel.any():
            print(f"critical-path runs with {lo}..{hi - 1} ops: {int(sel.sum())} runs, {int(pl[sel].sum())} ops, "
                  f"replay {prep[sel].sum() / 1e6:.3f} ms ({prep[sel].sum() / max(pl[sel].sum(), 1):.1f} ns/op)")
    for lo in (32, 1000, 10000):
        sel = rlen >= lo
        if sel.any():
            print(f"runs with >= {lo} ops: {int(sel.sum())}, {int(rlen[sel].sum())} ops, replay "
                  f"{(done - ready)[sel].sum() / rlen[sel].sum():.1f} ns/op")
    det = ready - np.maximum(dep_done, claim)
    print(f"all runs: median detect {np.median(det):.0f} ns, p90 {np.percentile(det, 90):.0f} ns; "
          f"median replay {np.median(done - ready):.0f} ns; claimed-after-ready fraction "
          f"{np.mean(claim > dep_done):.2f}")


if __name__ == "__main__":
    main()
