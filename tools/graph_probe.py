"""Small-batch apply latency: direct launches vs one CUDA-graph replay per batch.

usage: python tools/graph_probe.py [variant] [batch ...]
Prints one JSON line per batch size: per-batch device time for K batches
issued back to back on one stream (no host sync between batches), through
SfSketch._submit (the library's launches) and through a captured graph; the
final states are checked equal."""

import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1701_04148_b200 as P  # noqa: E402
from paper_1701_04148_b200 import _lib  # noqa: E402
from paper_1701_04148_b200._ops import normalize_stream  # noqa: E402

K = 200


def main():
    variant = sys.argv[1] if len(sys.argv) > 1 else "sff"
    sizes = [int(x) for x in sys.argv[2:]] or [1, 64, 1024, 16384]
    rng = np.random.default_rng(7)
    for b in sizes:
        keys = torch.as_tensor(rng.integers(0, 50_000, size=b, dtype=np.uint32)).cuda()
        ops = torch.zeros(b, dtype=torch.uint8, device="cuda")
        mk = lambda: P.SfSketch(P.SketchParams(d=4, w=65536, z=4, master_seed=2017), variant)  # noqa: E731
        ops_t, kb = normalize_stream(ops, keys)
        a, g_sk = mk(), mk()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            a._submit(ops_t, kb)
            g_sk._submit(ops_t, kb)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            g_sk._submit(ops_t, kb)
        out = {"variant": variant, "batch": b, "batches": K}
        for name, fn in (("direct", lambda: a._submit(ops_t, kb)), ("graph", g.replay)):
            fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(K):
                fn()
            e1.record()
            torch.cuda.synchronize()
            out[name + "_us_per_batch"] = round(e0.elapsed_time(e1) * 1e3 / K, 2)
        assert torch.equal(a.slim.counters, g_sk.slim.counters) and torch.equal(a.fat.counters, g_sk.fat.counters)
        out["speedup"] = round(out["direct_us_per_batch"] / out["graph_us_per_batch"], 2)
        L = _lib.lib()
        c0 = L.sfk_launch_count()
        a._submit(ops_t, kb)
        out["library_launches_per_batch"] = int(L.sfk_launch_count() - c0)  # CUB's sort launches not counted
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
