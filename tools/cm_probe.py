"""CM build timing (cfg 2: 10M inserts, d=4, w=65536): CUDA events around
CmSketch.apply_ops on device-resident inputs, median of 15; checked against
the oracle. Prints one JSON line. Usage: python tools/cm_probe.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1701_04148_b200 as P  # noqa: E402
from paper_1701_04148_b200 import workloads as W  # noqa: E402
from oracle import oracle as orc  # noqa: E402  (checker only)

c = W.cfg2(seed=2017)
ops, keys = torch.from_numpy(c["ops"]).cuda(), torch.from_numpy(c["keys"]).cuda()
ts = []
for r in range(18):
    cm = P.CmSketch(P.SketchParams(d=4, w=65536, master_seed=2017))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    cm.apply_ops(ops, keys)
    e1.record()
    torch.cuda.synchronize()
    if r >= 3:
        ts.append(e0.elapsed_time(e1))
o = orc.OracleSketch("cm", 4, 65536, master_seed=2017)
o.apply_ops(c["ops"], c["keys"].astype(np.uint64))
ok = bool(np.array_equal(cm.counters.cpu().numpy(), o.slim))
print(json.dumps({"cm_build_ms": round(float(np.median(ts)), 4), "equal_oracle": ok,
                  "lib": os.environ.get("SFK_LIB_PATH", "main")}), flush=True)
