"""Where the host time of a tiny SfSketch.apply_ops goes (1-op and 64-op
device batches): normalisation, the library call, the synchronising result
read. Prints one JSON line per batch size. Usage: python tools/api_overhead.py"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1701_04148_b200 as P  # noqa: E402
from paper_1701_04148_b200 import _lib  # noqa: E402
from paper_1701_04148_b200._ops import Scratch, normalize_stream  # noqa: E402

L = _lib.lib()
sk = P.SfSketch(P.SketchParams(d=4, w=65536, z=4, master_seed=1), "sff")
for n in (1, 64, 1024):
    ops = torch.zeros(n, dtype=torch.uint8, device="cuda")
    keys = torch.arange(n, dtype=torch.int64, device="cuda")
    R = 300
    for _ in range(20):
        sk.apply_ops(ops, keys)
    torch.cuda.synchronize()
    t = {"normalize": 0.0, "submit": 0.0, "read": 0.0, "total": 0.0}
    for _ in range(R):
        t0 = time.perf_counter()
        o, kb = normalize_stream(ops, keys, check_ops=False)
        t1 = time.perf_counter()
        res = sk._submit(o, kb)
        t2 = time.perf_counter()
        Scratch.read(res)
        t3 = time.perf_counter()
        t["normalize"] += t1 - t0
        t["submit"] += t2 - t1
        t["read"] += t3 - t2
    t0 = time.perf_counter()
    for _ in range(R):
        sk.apply_ops(ops, keys)
    t["total"] = time.perf_counter() - t0
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(R):
        sk._submit(o, kb)
    ev1.record()
    torch.cuda.synchronize()
    print(json.dumps({"batch": n, **{k: round(v / R * 1e6, 2) for k, v in t.items()},
                      "device_back_to_back_us": round(ev0.elapsed_time(ev1) * 1e3 / R, 2)}), flush=True)
