import sys, time, json
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_1701_04148_b200 as P
from paper_1701_04148_b200 import workloads as W
from paper_1701_04148_b200.sf import query_min_host
c = W.cfg3(seed=2017, alpha=1.0)
sk = P.SfSketch(P.SketchParams(d=4, w=65536, z=4, master_seed=2017), "sff")
sk.apply_ops(torch.from_numpy(c["ops"]).cuda(), torch.from_numpy(c["keys"]).cuda())
Q = 1_000_000_000
qk = torch.empty(Q, dtype=torch.uint32, device="cuda")
W.DeviceQueryStream(2022, c["distinct"], 1.0).keys(0, Q, out=qk)
qk_h = torch.empty(Q, dtype=torch.uint32).pin_memory(); qk_h.copy_(qk)
qo_h = torch.empty(Q, dtype=torch.int64).pin_memory()
for chunk, streams in ((1 << 25, 3), (1 << 24, 3), (1 << 26, 3), (1 << 25, 2), (1 << 25, 4), (1 << 23, 4)):
    ts = []
    for r in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        query_min_host(sk.slim.counters, sk._slim_seeds, qk_h, qo_h, chunk=chunk, streams=streams)
        torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    print(json.dumps({"chunk": chunk, "streams": streams, "ms": round(min(ts) * 1e3, 1)}), flush=True)
# raw PCIe: H2D 4 GB, D2H 8 GB alone and together
d_in = torch.empty(Q, dtype=torch.uint32, device="cuda"); d_out = torch.empty(Q, dtype=torch.int64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for name in ("h2d", "d2h", "both"):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    if name in ("h2d", "both"):
        with torch.cuda.stream(s1): d_in.copy_(qk_h, non_blocking=True)
    if name in ("d2h", "both"):
        with torch.cuda.stream(s2): qo_h.copy_(d_out, non_blocking=True)
    torch.cuda.synchronize(); print(json.dumps({name: round((time.perf_counter() - t0) * 1e3, 1)}), flush=True)
