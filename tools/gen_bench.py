"""Times workloads.generate on the GPU (CUDA events) against numpy's own
draws for the same spec on the host (the reference's generator is numpy +
numba). Usage: python tools/gen_bench.py"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1701_04148_b200 import workloads as W  # noqa: E402

for mode, n, v in (("none", 100_000_000, 1_000_000), ("interleaved", 10_000_000, 1_000_000),
                   ("interleaved", 10_000_000, 10_000)):
    spec = W.WorkloadSpec(kind="zipf", distinct_items=v, total_ops=n, zipf_skew=1.0, seed=11,
                          deletion_mode=mode, delete_prob=0.2)
    W.generate(spec)  # warm
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    wl = W.generate(spec)
    e1.record()
    torch.cuda.synchronize()
    gpu_ms = e0.elapsed_time(e1)
    t0 = time.perf_counter()
    rng = np.random.Generator(np.random.PCG64(11))
    cdf = np.cumsum(W.zipf_probabilities(v, 1.0))
    cdf[-1] = 1.0
    ranks = np.searchsorted(cdf, rng.random(n), side="right")
    host_ms = (time.perf_counter() - t0) * 1e3
    ok = bool(np.array_equal(ranks, wl.ranks.cpu().numpy())) if mode == "none" else None
    print(json.dumps({"mode": mode, "ops": n, "distinct": v, "gpu_ms": round(gpu_ms, 2),
                      "numpy_zipf_draws_ms": round(host_ms, 1), "ranks_equal": ok}))
