"""Engine counters for one cfg-3 SFF build (sfk_engine_stats): replay words by
path, replay cycles, runs, warp iterations, long-run pieces; plus the mean
warp-iteration time. Usage: python tools/engine_stats.py [alpha] [variant]"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1701_04148_b200 as P  # noqa: E402
from paper_1701_04148_b200 import _lib, workloads as W  # noqa: E402

alpha = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
variant = sys.argv[2] if len(sys.argv) > 2 else "sff"
L = _lib.lib()
c = W.cfg3(seed=2017, alpha=alpha)
ops, keys = torch.from_numpy(c["ops"]).cuda(), torch.from_numpy(c["keys"]).cuda()
P.SfSketch(P.SketchParams(d=4, w=65536, z=4, w_prime=262144, master_seed=2017), variant).apply_ops(ops, keys)
st = (ctypes.c_ulonglong * 8)()
L.sfk_engine_stats(st, 1)
L.sfk_engine_timing(1)
P.SfSketch(P.SketchParams(d=4, w=65536, z=4, w_prime=262144, master_seed=2017), variant).apply_ops(ops, keys)
ms = float(L.sfk_engine_last_ms())
L.sfk_engine_stats(st, 1)
sms = torch.cuda.get_device_properties(0).multi_processor_count
warps = sms * 8
names = ["gap_words", "steady_words", "general_words", "replay_cycles", "runs", "warp_iterations", "pieces", "piece_ops"]
out = dict(zip(names, [int(v) for v in st]))
out["engine_ms"] = round(ms, 3)
out["iterations_per_warp"] = round(out["warp_iterations"] / warps, 1)
out["ns_per_iteration"] = round(ms * 1e6 / max(out["warp_iterations"] / warps, 1), 1)
print(json.dumps(out))
