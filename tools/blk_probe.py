"""Phase timing of the block engine (sfk_blk.cu) on cfg-3-shaped SFF batches:
globaltimer stamps at its phase boundaries (sort, fat walk, dataflow replay,
write-back), read through the diagnostics symbol. Usage: python tools/blk_probe.py"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1701_04148_b200 as P  # noqa: E402
from paper_1701_04148_b200 import _lib, workloads as W  # noqa: E402

L = _lib.lib()

c = W.cfg3(seed=2017, n_ins=2_000_000, v=200_000, alpha=1.0)
ops_d, keys_d = torch.from_numpy(c["ops"]).cuda(), torch.from_numpy(c["keys"]).cuda()
buf = (ctypes.c_ulonglong * 6)()
for n in (64, 256, 512, 1024, 2048):
    sk = P.SfSketch(P.SketchParams(d=4, w=65536, z=4, master_seed=2017), "sff")
    acc = [0.0] * 5
    R = 50
    for b in range(R):
        sk.apply_ops(ops_d[b * n:(b + 1) * n], keys_d[b * n:(b + 1) * n])
        torch.cuda.synchronize()
        L.sfk_blk_profile(buf)
        for k in range(5):
            acc[k] += (buf[k + 1] - buf[k]) / 1e3
    print(json.dumps({"batch": n, "us": dict(zip(["hash_sort", "scan", "fat_pass", "replay", "write_back"],
                                                   [round(x / R, 2) for x in acc]))}), flush=True)
