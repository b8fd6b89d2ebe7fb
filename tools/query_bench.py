"""cfg-5 query sweep: the slim built from the cfg-3 stream (alpha = 1.0), then
Q point queries (50% present with Zipf(alpha_q) rank skew, 50% absent) for
alpha_q in 0.0 .. 3.0, timed per kernel path (L2 gathers / row-partitioned
cluster) with CUDA events on the launching stream, L2 flushed between reps.
Every path's estimates are checked equal to the L2 path's over the full batch,
and a 2M-key sample against the CPU oracle.
Usage: python tools/query_bench.py [Q] [alphas comma-separated] [paths comma-separated]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1701_04148_b200 as P  # noqa: E402
from paper_1701_04148_b200 import _lib, workloads as W  # noqa: E402

Q = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000_000
ALPHAS = [float(a) for a in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0.0, 0.5, 1.0, 1.5, 2.0, 2.5, 3.0]
PATHS = [int(p) for p in sys.argv[3].split(",")] if len(sys.argv) > 3 else [1, 3]
KEYS64 = len(sys.argv) > 4 and sys.argv[4] == "u64"
NAMES = {1: "l2", 2: "smem", 3: "cluster", 4: "cw"}
REPS = 5

L = _lib.lib()
dev = torch.device("cuda", 0)
c = W.cfg3(seed=2017, alpha=1.0)
sk = P.SfSketch(P.SketchParams(d=4, w=65536, z=4, master_seed=2017), "sff")
sk.apply_ops(torch.from_numpy(c["ops"]).to(dev), torch.from_numpy(c["keys"]).to(dev))
slim = sk.slim.counters
seeds = sk._slim_seeds
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
keys = torch.empty(Q, dtype=torch.uint32, device=dev)
ref = torch.empty(Q, dtype=torch.int64, device=dev)
out = torch.empty(Q, dtype=torch.int64, device=dev)
from oracle import oracle as orc  # noqa: E402  (checker only)

slim_h = slim.cpu().numpy()


keys64 = torch.empty(Q, dtype=torch.int64, device=dev) if KEYS64 else None


def run(path, o):
    prev = L.sfk_query_path(path)
    kp, kind = (keys64.data_ptr(), _lib.KEY_U64) if KEYS64 else (keys.data_ptr(), _lib.KEY_U32)
    rc = L.sfk_min_query(slim.data_ptr(), seeds.ctypes.data, 4, 65536, kp, kind, 0, Q,
                         o.data_ptr(), _lib.stream_ptr())
    L.sfk_query_path(prev)
    _lib.check(rc, "sfk_min_query")
    return L.sfk_query_last_path()


for aq in ALPHAS:
    W.DeviceQueryStream(2017 + 5, c["distinct"], aq).keys(0, Q, out=keys)
    if KEYS64:
        keys64.copy_(keys.to(torch.int64))  # the same keys, zero-extended (estimates are identical)
    torch.cuda.synchronize()
    for p in PATHS:
        o = ref if p == PATHS[0] else out
        took = run(p, o)  # warm
        times = []
        for _ in range(REPS):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            run(p, o)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        ms = float(np.median(times))
        same = True if o is ref else bool(torch.equal(out, ref))
        sample = keys[:2_000_000].cpu().numpy().astype(np.uint64)
        ok_oracle = bool(np.array_equal(o[:2_000_000].cpu().numpy(), orc.min_query(slim_h, seeds, sample, threads=8)))
        print(json.dumps({"alpha_q": aq, "keys": "u64" if KEYS64 else "u32", "path": NAMES[took], "queries": Q,
                          "ms": round(ms, 3),
                          "Gq_s": round(Q / ms / 1e6, 2), "hbm_GBps_12B": round(Q * 12 / ms / 1e6, 1),
                          "equal_to_first_path": same, "oracle_sample_2M_equal": ok_oracle}), flush=True)
        assert same and ok_oracle
