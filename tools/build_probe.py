"""Times one SF build (CUDA events, median of REPS) and the engine kernel
alone (sfk_engine_timing); prints one JSON line. Diagnostics for engine
knobs set through the environment (SFK_ENGINE_BUDGET, SFK_ENGINE_BLOCKS_PER_SM).
Usage: python tools/build_probe.py [variant] [alpha] [cfg]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1701_04148_b200 as P  # noqa: E402
from paper_1701_04148_b200 import _lib, workloads as W  # noqa: E402

variant = sys.argv[1] if len(sys.argv) > 1 else "sff"
alpha = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
cfg = sys.argv[3] if len(sys.argv) > 3 else "3"
L = _lib.lib()
dev = torch.device("cuda", 0)
if variant == "cu":
    c = W.cfg2(seed=2017)
    ops, keys = torch.from_numpy(c["ops"]).to(dev), torch.from_numpy(c["keys"]).to(dev)
    params = P.SketchParams(d=4, w=65536, master_seed=2017)
elif cfg == "1":
    c = W.cfg1(seed=2017)
    ops, keys = torch.from_numpy(c["ops"]).to(dev), torch.from_numpy(c["keys"]).to(dev)
    params = P.SketchParams(d=4, w=16384, w_prime=65536, master_seed=2017)
elif cfg == "4":
    c = W.cfg4(seed=2017)
    ops, keys = torch.from_numpy(c["ops"]).to(dev), torch.from_numpy(c["records"]).to(dev)
    params = P.SketchParams(d=4, w=12800, w_prime=4194304, master_seed=2017)
else:
    c = W.cfg3(seed=2017, alpha=alpha)
    ops, keys = torch.from_numpy(c["ops"]).to(dev), torch.from_numpy(c["keys"]).to(dev)
    params = P.SketchParams(d=4, w=65536, z=4, w_prime=262144, master_seed=2017)
ts, es = [], []
L.sfk_engine_timing(1)
for r in range(6):
    sk = P.CuSketch(params) if variant == "cu" else P.SfSketch(params, variant)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sk.apply_ops(ops, keys)
    e1.record()
    torch.cuda.synchronize()
    if r:
        ts.append(e0.elapsed_time(e1))
        es.append(float(L.sfk_engine_last_ms()))
print(json.dumps({"variant": variant, "alpha": alpha, "cfg": cfg, "env": {k: v for k, v in os.environ.items()
                  if k.startswith("SFK_")}, "build_ms": round(float(np.median(ts)), 3),
                  "engine_ms": round(float(np.median(es)), 3)}), flush=True)
