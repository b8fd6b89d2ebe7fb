"""Run the cfg-3 SFF build (and optionally other configs) a few times; used
under `ncu --metrics gpu__time_duration.sum` to get the per-kernel launch list
of one apply_ops call. Usage: python tools/one_build.py [sff|sf1|cu|cm|sf1rec] [alpha] [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1701_04148_b200 as P  # noqa: E402
from paper_1701_04148_b200 import workloads as W  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "sff"
alpha = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
if kind == "sff":
    c = W.cfg3(seed=2017, alpha=alpha)
    params, keys = P.SketchParams(d=4, w=65536, z=4, master_seed=2017), c["keys"]
elif kind == "sf1":
    c = W.cfg1(seed=2017)
    params, keys = P.SketchParams(d=4, w=16384, z=4, master_seed=2017), c["keys"]
elif kind == "sf1rec":
    c = W.cfg4(seed=2017, n=int(sys.argv[4]) if len(sys.argv) > 4 else 100_000_000)
    params, keys = P.SketchParams(d=4, w=12800, w_prime=4194304, master_seed=2017), c["records"]
else:
    c = W.cfg2(seed=2017)
    params, keys = P.SketchParams(d=4, w=65536, master_seed=2017), c["keys"]
ops_d = torch.from_numpy(c["ops"]).cuda()
keys_d = torch.from_numpy(keys).cuda()
for r in range(reps):
    if kind in ("cm", "cu"):
        sk = P.CmSketch(params) if kind == "cm" else P.CuSketch(params)
    else:
        sk = P.SfSketch(params, "sf1" if kind.startswith("sf1") else "sff")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sk.apply_ops(ops_d, keys_d)
    torch.cuda.synchronize()
    print(f"{kind} alpha={alpha} rep {r}: {(time.perf_counter() - t0) * 1e3:.2f} ms for {len(c['ops'])} ops", flush=True)
import ctypes  # noqa: E402
from paper_1701_04148_b200 import _lib  # noqa: E402
st = (ctypes.c_ulonglong * 8)()
_lib.load_library().sfk_engine_stats(st, 1)
print("engine stats (all reps): gap_words=%d steady_words=%d slow_words=%d replay_cycles=%d runs=%d warp_iters=%d longrun_pieces=%d longrun_ops=%d" % tuple(st[:8]))
