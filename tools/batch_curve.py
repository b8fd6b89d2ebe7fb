"""Query batch-size curve (the paper's only GPU result,
PAPER.md:1413-1420: ~50 Mqps at 20K-query batches, >110 Mqps at 64K, latency
under 410 us). The cfg-3 (alpha = 1.0) SFF slim, cfg-5 query keys
(alpha_q = 1.0); per batch size:
  * device: keys already in HBM, one sfk_min_query per batch back to back
    (CUDA events over REPS batches) -> Mqps and us per batch;
  * host: each batch from pinned host memory through the public API path
    (H2D copy, kernel, D2H copy of the int64 estimates, then a host sync):
    the latency a caller sees per batch, and the rate of a closed loop.
Every batch size's estimates are checked against the oracle on a sample.
Prints one JSON line per batch size. Usage: python tools/batch_curve.py"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1701_04148_b200 as P  # noqa: E402
from paper_1701_04148_b200 import _lib, workloads as W  # noqa: E402

SIZES = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [
    1_000, 20_000, 64_000, 256_000, 1_000_000, 4_000_000, 16_000_000, 64_000_000]
L = _lib.lib()
dev = torch.device("cuda", 0)
c = W.cfg3(seed=2017, alpha=1.0)
sk = P.SfSketch(P.SketchParams(d=4, w=65536, z=4, master_seed=2017), "sff")
sk.apply_ops(torch.from_numpy(c["ops"]).to(dev), torch.from_numpy(c["keys"]).to(dev))
slim, seeds = sk.slim.counters, sk._slim_seeds
from oracle import oracle as orc  # noqa: E402  (checker only)

o = orc.OracleSketch("sff", 4, 65536, 4, None, 2017)
o.apply_ops(c["ops"], c["keys"].astype(np.uint64))
maxn = max(SIZES)
keys_d = W.DeviceQueryStream(2017 + 5, c["distinct"], 1.0).keys(0, maxn)
keys_h = torch.empty(maxn, dtype=torch.uint32).pin_memory()
keys_h.copy_(keys_d)
out_d = torch.empty(maxn, dtype=torch.int64, device=dev)
out_h = torch.empty(maxn, dtype=torch.int64).pin_memory()
kbuf = torch.empty(maxn, dtype=torch.uint32, device=dev)
st = torch.cuda.current_stream()


def q(kt, n, ot):
    _lib.check(L.sfk_min_query(slim.data_ptr(), seeds.ctypes.data, 4, 65536, kt.data_ptr(), _lib.KEY_U32, 0, n,
                               ot.data_ptr(), _lib.stream_ptr()), "sfk_min_query")


for n in SIZES:
    reps = max(3, min(2000, int(2e8 // n)))
    nb = maxn // n
    # device-resident: back-to-back batches over distinct slices of the keys
    for i in range(3):
        q(keys_d[(i % nb) * n:], n, out_d[(i % nb) * n:])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(reps):
        q(keys_d[(i % nb) * n:], n, out_d[(i % nb) * n:])
    e1.record()
    torch.cuda.synchronize()
    dev_us = e0.elapsed_time(e1) * 1e3 / reps
    path = int(L.sfk_query_last_path())
    # host round trip per batch (closed loop: one batch in flight)
    hreps = max(3, min(500, int(5e7 // n)))
    lat = []
    for i in range(hreps + 2):
        a = (i % nb) * n
        t0 = time.perf_counter()
        kbuf[:n].copy_(keys_h[a:a + n], non_blocking=True)
        q(kbuf, n, out_d)
        out_h[a:a + n].copy_(out_d[:n], non_blocking=True)
        st.synchronize()
        if i >= 2:
            lat.append(time.perf_counter() - t0)
    lat_us = float(np.median(lat)) * 1e6
    m = min(n, 2_000_000)
    ok = bool(np.array_equal(out_h[:m].numpy(), o.query_many(keys_h[:m].numpy().astype(np.uint64), threads=8)))
    print(json.dumps({"batch": n, "path": {1: "l2", 2: "smem", 3: "cluster", 4: "cw"}.get(path, path),
                      "device_us_per_batch": round(dev_us, 2), "device_Mqps": round(n / dev_us, 1),
                      "host_roundtrip_us_median": round(lat_us, 1), "host_closed_loop_Mqps": round(n / lat_us, 1),
                      "oracle_equal": ok}), flush=True)
    assert ok
