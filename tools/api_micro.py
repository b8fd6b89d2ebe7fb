"""Host-side cost of the pieces of one tiny SfSketch.apply_ops (device-resident
inputs): library lookup, device(), normalisation, workspace query, scratch,
stream handle, the C call (launch included), the synchronising read.
Prints one JSON line of microseconds per call. Usage: python tools/api_micro.py"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1701_04148_b200 as P  # noqa: E402
from paper_1701_04148_b200 import _lib  # noqa: E402
from paper_1701_04148_b200._ops import Scratch, device, normalize_stream  # noqa: E402

L = _lib.lib()
sk = P.SfSketch(P.SketchParams(d=4, w=65536, z=4, master_seed=1), "sff")
ops = torch.zeros(1, dtype=torch.uint8, device="cuda")
keys = torch.arange(1, dtype=torch.int64, device="cuda")
R = 2000


def t(fn):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(R):
        fn()
    torch.cuda.synchronize()
    return round((time.perf_counter() - t0) / R * 1e6, 2)


o, kb = normalize_stream(ops, keys, check_ops=False)
res = sk._submit(o, kb)
out = {
    "lib": t(lambda: _lib.lib()),
    "device": t(lambda: device()),
    "normalize": t(lambda: normalize_stream(ops, keys, check_ops=False)),
    "workspace_size": t(lambda: L.sfk_sf_workspace_size(6, 4, 65536, 0, 4, 1)),
    "scratch_get": t(lambda: sk._scratch.get(256)),
    "stream_ptr": t(lambda: _lib.stream_ptr()),
    "data_ptr_x7": t(lambda: [sk.slim.counters.data_ptr() for _ in range(7)]),
    "submit": t(lambda: sk._submit(o, kb)),
    "submit_read": t(lambda: Scratch.read(sk._submit(o, kb))),
    "apply_ops": t(lambda: sk.apply_ops(ops, keys)),
    "insert": t(lambda: sk.insert(5)),
}
print(json.dumps(out), flush=True)
