"""Two-phase query timing (diagnostics): the cfg-3 build, the 1B-key index
pass, the gather pass, and the build with the index pass running beside it on
a second stream. CUDA events; prints one JSON line."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1701_04148_b200 as P  # noqa: E402
from paper_1701_04148_b200 import _lib, workloads as W  # noqa: E402

Q = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000_000
L = _lib.lib()
dev = torch.device("cuda", 0)
c = W.cfg3(seed=2017, alpha=1.0)
ops, keys = torch.from_numpy(c["ops"]).to(dev), torch.from_numpy(c["keys"]).to(dev)
qk = torch.empty(Q, dtype=torch.uint32, device=dev)
W.DeviceQueryStream(2022, c["distinct"], 1.0).keys(0, Q, out=qk)
idx = torch.empty(4 * Q, dtype=torch.uint16, device=dev)
out = torch.empty(Q, dtype=torch.int64, device=dev)
ref = torch.empty(Q, dtype=torch.int64, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
sk = P.SfSketch(P.SketchParams(d=4, w=65536, z=4, master_seed=2017), "sff")
seeds = sk._slim_seeds.ctypes.data_as(ctypes.c_void_p)
side = torch.cuda.Stream()


def reset():
    sk.slim.counters.zero_()
    sk.fat.counters.zero_()
    sk.slim.increment_counts.zero_()
    sk.slim.insertions_seen = 0


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


def run(fn, reps=4):
    ts = []
    for _ in range(reps + 1):
        flush.fill_(1)
        torch.cuda.synchronize()
        e0 = ev()
        fn()
        e1 = ev()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts[1:]))


def build():
    reset()
    sk.apply_ops(ops, keys)


def index(stream=None):
    _lib.check(L.sfk_query_index(seeds, 4, 65536, qk.data_ptr(), _lib.KEY_U32, 0, Q, idx.data_ptr(),
                                 _lib.stream_ptr(stream)), "index")


def gather():
    _lib.check(L.sfk_min_query_idx(sk.slim.counters.data_ptr(), 4, 65536, idx.data_ptr(), Q, out.data_ptr(),
                                   _lib.stream_ptr()), "gather")


def fused():
    _lib.check(L.sfk_min_query(sk.slim.counters.data_ptr(), sk._slim_seeds.ctypes.data, 4, 65536, qk.data_ptr(),
                               _lib.KEY_U32, 0, Q, ref.data_ptr(), _lib.stream_ptr()), "fused")


def overlapped():
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        index(side)
    build()
    torch.cuda.current_stream().wait_stream(side)
    gather()


if len(sys.argv) > 2 and sys.argv[2] == "gather":  # for ncu: one build, one index, one gather
    build()
    index()
    gather()
    torch.cuda.synchronize()
    sys.exit(0)
r = {"queries": Q}
r["build_ms"] = run(build)
r["fused_query_ms"] = run(fused)
r["index_ms"] = run(index)
r["gather_ms"] = run(gather)
r["build_plus_fused_ms"] = round(r["build_ms"] + r["fused_query_ms"], 3)
r["overlapped_step_ms"] = run(overlapped)
r["equal"] = bool(torch.equal(out, ref))
print(json.dumps(r))
