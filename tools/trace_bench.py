"""Trace ingestion speed: a 5M-line "OP,key" trace parsed on the GPU
(workloads.load_trace) against the reference's per-line rules run in Python
on the host over a 500k-line sample. Usage: python tools/trace_bench.py"""
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1701_04148_b200 import workloads as W  # noqa: E402

n = 5_000_000
rng = np.random.default_rng(1)
keys = rng.integers(0, np.iinfo(np.uint64).max, size=n, dtype=np.uint64)
ops = (rng.random(n) < 0.2).astype(np.uint8)
path = os.path.join(tempfile.mkdtemp(), "bench.trace")
with open(path, "w") as fh:
    fh.write("".join(f"{'D' if o else 'I'},{k}\n" for o, k in zip(ops, keys)))
size = os.path.getsize(path)
W.load_trace(path)  # warm
torch.cuda.synchronize()
t0 = time.perf_counter()
o, k = W.load_trace(path)
torch.cuda.synchronize()
gpu_s = time.perf_counter() - t0
ok = bool(np.array_equal(o.cpu().numpy(), ops) and np.array_equal(k.cpu().numpy(), keys))
sample = 500_000
t0 = time.perf_counter()
with open(path, "r", encoding="utf-8") as fh:
    for i, line in enumerate(fh, start=1):
        W._trace_line(line, i)
        if i == sample:
            break
host_s = (time.perf_counter() - t0) * n / sample
print(json.dumps({"lines": n, "bytes": size, "gpu_load_trace_s": round(gpu_s, 3),
                  "gpu_GB_s_incl_file_read": round(size / gpu_s / 1e9, 2),
                  "host_python_rules_s_extrapolated": round(host_s, 2), "equal": ok}))
