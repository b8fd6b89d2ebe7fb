"""Times one big batch against the same ops applied as consecutive slices
(the chunked results are identical by the batch semantics); for choosing the
C ABI's internal chunk size. Usage: python tools/chunk_probe.py [sf1rec|sff|cu]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1701_04148_b200 as P  # noqa: E402
from paper_1701_04148_b200 import workloads as W  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "sf1rec"
if kind == "sf1rec":
    c = W.cfg4(seed=2017)
    ops, keys = torch.from_numpy(c["ops"]).cuda(), torch.from_numpy(c["records"]).cuda()
    mk = lambda: P.SfSketch(P.SketchParams(d=4, w=12800, w_prime=4194304, master_seed=2017), "sf1")  # noqa: E731
elif kind == "cu":
    c = W.cfg2(seed=2017)
    ops, keys = torch.from_numpy(c["ops"]).cuda(), torch.from_numpy(c["keys"]).cuda()
    mk = lambda: P.CuSketch(P.SketchParams(d=4, w=65536, master_seed=2017))  # noqa: E731
else:
    c = W.cfg3(seed=2017, alpha=1.0)
    ops, keys = torch.from_numpy(c["ops"]).cuda(), torch.from_numpy(c["keys"]).cuda()
    mk = lambda: P.SfSketch(P.SketchParams(d=4, w=65536, z=4, master_seed=2017), "sff")  # noqa: E731
n = ops.numel()
ref = None
for parts in (1, 2, 4, 8, 16):
    ts = []
    for r in range(3):
        sk = mk()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        b = np.linspace(0, n, parts + 1).astype(int)
        for a, z in zip(b[:-1], b[1:]):
            sk.apply_ops(ops[a:z], keys[a:z])
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    cnt = (sk.slim.counters if hasattr(sk, "slim") else sk.counters).cpu().numpy()
    ref = cnt if ref is None else ref
    print(json.dumps({"kind": kind, "parts": parts, "ms": round(min(ts), 2), "same": bool(np.array_equal(cnt, ref))}),
          flush=True)
