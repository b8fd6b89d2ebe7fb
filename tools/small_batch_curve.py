"""Per-batch latency of SfSketch("sff").apply_ops through the public API
(device-resident ops/keys, the result triple read back each batch, as the
API does) for small batch sizes, on each engine: the warp-cooperative exact
engine (sfk_warp_batch_ops), the one-CTA block engine (sfk_block_batch_ops,
up to 8192 (op, row) pairs), the one-thread engine (sfk_small_batch_ops)
and the parallel pipeline; plus "auto" (the library's defaults); beside the reference (numba, baseline/_ref) and
the C port on one host thread over the same batches. VERDICT r01 item 7:
a 64-op SFF batch under 60 us, and the GPU ahead of one CPU thread from 1K
ops. Prints one JSON line per batch size. Usage: python tools/small_batch_curve.py"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1701_04148_b200 as P  # noqa: E402
from paper_1701_04148_b200 import _lib, workloads as W  # noqa: E402
from oracle import oracle as orc  # noqa: E402  (CPU baseline)

SIZES = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [1, 8, 64, 256, 512, 1024, 2048, 4096, 16384]
L = _lib.lib()
c = W.cfg3(seed=2017, n_ins=2_000_000, v=200_000, alpha=1.0)
ops_h, keys_h = c["ops"], c["keys"]
ops_d, keys_d = torch.from_numpy(ops_h).cuda(), torch.from_numpy(keys_h).cuda()
ref = bench.ref_package()
params = P.SketchParams(d=4, w=65536, z=4, master_seed=2017)


def gpu_run(n, mode, batches):
    prev_s, prev_w, prev_b = L.sfk_small_batch_ops(-1), L.sfk_warp_batch_ops(-1), L.sfk_block_batch_ops(-1)
    if mode != "auto":
        L.sfk_small_batch_ops(32 if mode == "one-thread" else 0)
        L.sfk_warp_batch_ops(1 << 30 if mode == "warp" else 0)
        L.sfk_block_batch_ops(1 << 30 if mode == "block" else 0)
    try:
        sk = P.SfSketch(params, "sff")
        sk.apply_ops(ops_d[:n], keys_d[:n])  # warm
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for b in range(1, batches + 1):
            sk.apply_ops(ops_d[b * n:(b + 1) * n], keys_d[b * n:(b + 1) * n])
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / batches * 1e6
    finally:
        L.sfk_small_batch_ops(prev_s)
        L.sfk_warp_batch_ops(prev_w)
        L.sfk_block_batch_ops(prev_b)


for n in SIZES:
    batches = max(5, min(200, 400_000 // n))
    row = {"batch": n, "batches": batches}
    for mode in ("auto", "warp", "block", "one-thread", "parallel"):
        if (mode == "one-thread" and n > 4096) or (mode == "warp" and n > 4096) or (mode == "block" and n > 2048):
            continue
        row[f"{mode}_us"] = round(gpu_run(n, mode, batches), 1)
    o = orc.OracleSketch("sff", 4, 65536, 4, None, 2017)
    k64 = keys_h.astype(np.uint64)
    t0 = time.perf_counter()
    for b in range(0, batches):
        o.apply_ops(ops_h[b * n:(b + 1) * n], k64[b * n:(b + 1) * n])
    row["cpu_port_us"] = round((time.perf_counter() - t0) / batches * 1e6, 1)
    if ref is not None:
        r = ref.SfSketch(ref.SketchParams(d=4, w=65536, z=4, master_seed=2017), "sff")
        ref.SfSketch(ref.SketchParams(d=4, w=65536, z=4, master_seed=2017), "sff").apply_ops(ops_h[:1], k64[:1])  # compile
        t0 = time.perf_counter()
        for b in range(0, batches):
            r.apply_ops(ops_h[b * n:(b + 1) * n], k64[b * n:(b + 1) * n])
        row["reference_us"] = round((time.perf_counter() - t0) / batches * 1e6, 1)
    print(json.dumps(row), flush=True)
