"""Synthetic-stream fixtures: what the REFERENCE's workloads.generate makes of
a set of specs (build container only; imports /root/reference):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_workloads.py

Writes tests/golden/streams/workloads.npz: per case the spec fields and the
reference's ops / ranks (its keys are finalize64 of the ranks).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from sfsketch.workloads import WorkloadSpec, generate  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def _finalize(r):
    from sfsketch.hashing import finalize64_array

    return finalize64_array(r.astype(np.uint64))

CASES = [
    ("zipf_none", dict(kind="zipf", distinct_items=1000, total_ops=50_000, zipf_skew=0.99, seed=1)),
    ("zipf_reverse", dict(kind="zipf", distinct_items=300, total_ops=20_000, zipf_skew=1.3, seed=2,
                          deletion_mode="reverse_order")),
    ("zipf_interleaved", dict(kind="zipf", distinct_items=2000, total_ops=60_000, zipf_skew=0.8, seed=3,
                              deletion_mode="interleaved", delete_prob=0.3)),
    ("zipf_one_item", dict(kind="zipf", distinct_items=1, total_ops=1000, zipf_skew=2.0, seed=4)),
    ("zipf_empty", dict(kind="zipf", distinct_items=50, total_ops=0, seed=5)),
    ("uniform_none", dict(kind="uniform", distinct_items=777, total_ops=30_000, seed=6)),
    ("uniform_interleaved", dict(kind="uniform", distinct_items=100, total_ops=30_000, seed=7,
                                 deletion_mode="interleaved", delete_prob=0.45)),
    ("zipf_big_seed", dict(kind="zipf", distinct_items=100_000, total_ops=200_000, zipf_skew=1.1,
                           seed=2**63 + 12345, deletion_mode="interleaved", delete_prob=0.2)),
]


def main():
    out = {}
    meta = {}
    for name, spec in CASES:
        wl = generate(WorkloadSpec(**spec))
        out[name + "_ops"] = wl.ops
        out[name + "_ranks"] = wl.ranks
        assert np.array_equal(wl.keys, _finalize(wl.ranks))  # keys = finalize64(rank): not stored
        meta[name] = spec
    out["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    os.makedirs(os.path.join(OUT, "streams"), exist_ok=True)
    np.savez_compressed(os.path.join(OUT, "streams", "workloads.npz"), **out)
    print({k: len(out[k + "_ops"]) for k in meta})


if __name__ == "__main__":
    main()
