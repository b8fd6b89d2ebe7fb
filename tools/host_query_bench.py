"""Host-buffer query sweep (sfk_min_query_host, DESIGN.md §5 e2e): the cfg-3
alpha = 1.0 slim, Q cfg-5 keys (alpha_q = 1.0) in host memory, estimates into
a host int64 array, wall-clocked per call (3 reps, best and mean) for each
wire format / chunk size / direct-chunk share / ring depth given, with pinned
or pageable buffers. Every configuration's output is checked equal to the
device-resident query_many over the whole batch.
Usage: python tools/host_query_bench.py [Q] [spec ...]
  spec = wire:chunk_log2:direct:ring:mem[:threads]   (wire 1 i64 / 2 u32 /
         3 c16; mem p = pinned keys+out, g = pageable keys+out, k = pageable
         keys only; threads 0 = the library default)"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1701_04148_b200 as P  # noqa: E402
from paper_1701_04148_b200 import _lib, workloads as W  # noqa: E402
from paper_1701_04148_b200.sf import query_min_host  # noqa: E402

Q = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000_000
SPECS = sys.argv[2:] or ["1:25:0:3:p", "2:24:0:4:p", "3:24:0:4:p", "3:24:3:4:p", "3:24:4:4:p"]
L = _lib.lib()
dev = torch.device("cuda", 0)
c = W.cfg3(seed=2017, alpha=1.0)
sk = P.SfSketch(P.SketchParams(d=4, w=65536, z=4, master_seed=2017), "sff")
sk.apply_ops(torch.from_numpy(c["ops"]).to(dev), torch.from_numpy(c["keys"]).to(dev))
keys_d = W.DeviceQueryStream(2017 + 5, c["distinct"], 1.0).keys(0, Q)
ref = sk.query_many(keys_d)
torch.cuda.synchronize()
kp = keys_d.cpu().pin_memory()
op = torch.empty(Q, dtype=torch.int64).pin_memory()
kg = None
og = None
print(json.dumps({"probe": "setup", "queries": Q, "threads": os.cpu_count()}), flush=True)
for spec in SPECS:
    f = spec.split(":") + ["0"]
    wire, clog, direct, ring, mem, threads = f[:6]
    L.sfk_host_query_config(_lib.HQ_THREADS, int(threads))
    L.sfk_host_query_config(_lib.HQ_WIRE, int(wire))
    L.sfk_host_query_config(_lib.HQ_CHUNK, 1 << int(clog))
    L.sfk_host_query_config(_lib.HQ_DIRECT, int(direct))
    L.sfk_host_query_config(_lib.HQ_RING, int(ring))
    if mem in "gk" and kg is None:
        kg = torch.from_numpy(kp.numpy().copy())
    if mem == "g" and og is None:
        og = torch.from_numpy(np.ones(Q, np.int64))  # touched: no first-touch faults in the timed call
    k = kp if mem == "p" else kg
    o = op if mem in "pk" else og
    ts = []
    for rep in range(4):
        o.fill_(-1) if rep == 0 else None
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        query_min_host(sk.slim.counters, sk._slim_seeds, k, o)
        ts.append(time.perf_counter() - t0)
    ok = torch.equal(o.to(dev), ref)
    ts = ts[1:]
    print(json.dumps({"spec": spec, "wire_used": int(L.sfk_host_query_config(_lib.HQ_LAST_WIRE, -1)),
                      "best_ms": round(min(ts) * 1e3, 2), "mean_ms": round(sum(ts) / len(ts) * 1e3, 2),
                      "Gq_s": round(Q / min(ts) / 1e9, 3), "equal": bool(ok)}), flush=True)
