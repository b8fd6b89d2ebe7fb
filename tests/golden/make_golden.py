"""Regenerate the golden fixtures by running the REFERENCE implementation.

Run in the build container only (it imports /root/reference, which does not
exist on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Every fixture records the inputs (params, ops, keys, any preset state) and
the reference's outputs (slim/fat/deletion counters, tallies,
insertions_seen, status/op_index/n_ins of apply_ops, query estimates, the
export payload). The tests replay the inputs through the CPU oracle and
through the CUDA path and demand bit-identical results.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from sfsketch import (  # noqa: E402
    CmSketch,
    CuSketch,
    SfSketch,
    SketchParams,
    export_slim,
)
from sfsketch import _kernels  # noqa: E402
from sfsketch import hashing as H  # noqa: E402
from sfsketch.workloads import WorkloadSpec, generate  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
STATUS = {"PhantomDeletionError": 1, "SaturationError": 2, "UnsupportedOperationError": 3}


def make(kind, params):
    if kind == "cm":
        return CmSketch(params)
    if kind == "cu":
        return CuSketch(params)
    return SfSketch(params, kind)


def state(sk):
    if isinstance(sk, SfSketch):
        out = {"slim": sk.slim.counters.copy(), "inc": sk.slim.increment_counts.copy(),
               "seen": np.int64(sk.slim.insertions_seen), "fat": sk.fat.counters.copy()}
        if sk.deletion_sub is not None:
            out["dsub"] = sk.deletion_sub.counters.copy()
        return out
    return {"slim": sk.counters.copy(), "inc": sk.increment_counts.copy(), "seen": np.int64(sk.insertions_seen)}


def run_case(name, kind, params, ops, keys, preset=None, query_keys=None, batches=1):
    sk = make(kind, params)
    if preset:
        for attr, val in preset.items():
            if attr == "fat":
                sk.fat.counters[...] = val
            elif attr == "slim":
                (sk.slim.counters if isinstance(sk, SfSketch) else sk.counters)[...] = val
    before = {f"pre_{k}": v for k, v in state(sk).items()}
    status, op_index = 0, -1
    bounds = np.linspace(0, len(ops), batches + 1).astype(int)
    for a, b in zip(bounds[:-1], bounds[1:]):
        try:
            sk.apply_ops(ops[a:b], keys[a:b])
        except Exception as e:  # noqa: BLE001 - the reference's status exceptions
            status = STATUS[type(e).__name__]
            op_index = a + int(str(e).split(":")[0].split()[1])
            break
    if query_keys is None:
        query_keys = np.unique(keys)[:4096]
    q = sk.query_many(query_keys)
    fx = {"kind": np.array(kind), "d": np.int64(params.d), "w": np.int64(params.w), "z": np.int64(params.z),
          "w_prime": np.int64(params.w_prime), "master_seed": np.uint64(params.master_seed),
          "ops": np.ascontiguousarray(ops, dtype=np.uint8), "keys": np.ascontiguousarray(keys),
          "batches": np.int64(batches), "status": np.int64(status), "op_index": np.int64(op_index),
          "query_keys": np.ascontiguousarray(query_keys), "query": q,
          "export": np.frombuffer(export_slim(sk), dtype=np.uint8)}
    fx.update(before)
    fx.update(state(sk))
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **fx)
    return status, op_index


def mixed_stream(seed, n, v, p, alpha=1.0):
    wl = generate(WorkloadSpec(kind="zipf", distinct_items=v, total_ops=n, zipf_skew=alpha, seed=seed,
                               deletion_mode="interleaved", delete_prob=p))
    return wl.ops, wl.keys


def main():
    manifest = {}
    # ---------------------------------------------------------------- hashing
    finals = [0, 1, 2, 0x2A, 0x123456789ABCDEF0, 0xFFFFFFFFFFFFFFFF, 0x9E3779B97F4A7C15]
    rng = np.random.Generator(np.random.PCG64(7))
    many = rng.integers(0, 1 << 63, size=256, dtype=np.uint64) * np.uint64(2) + np.uint64(1)
    mixed = np.empty(many.shape[0], dtype=np.uint64)
    _kernels.mix_batch(many, mixed)
    strings = ["", "apple", "apples", "flow:10.0.0.1:80", "été", "x" * 13]
    hashing = {
        "finalize": {str(x): str(H.finalize64(x)) for x in finals},
        "mix_batch_in": [str(int(x)) for x in many],
        "mix_batch_out": [str(int(x)) for x in mixed],
        "seeds": {f"{m}:{d}": [str(s) for s in H.derive_seeds(m, d).per_array_seeds] for m, d in
                  [(0, 1), (0, 4), (5, 3), (2017, 8), (0xFFFFFFFFFFFFFFFF, 4)]},
        "seed_array_ext": {f"{m}:{d}": [str(int(s)) for s in H.seed_array(m, d, d)] for m, d in [(0, 4), (2017, 4)]},
        "key_from_string": {s: str(H.key_from_string(s)) for s in strings},
        "bucket": [[str(k), i, r, H.bucket_hash(H.derive_seeds(6, 4), i, k, r)]
                   for k in [0, 1, 42, 2**63 + 5, 2**64 - 1] for i in range(4) for r in [1, 13, 12800, 65536]],
        "slot": [[str(k), i, z, H.slot_hash(H.derive_seeds(6, 4), i, k, z)]
                 for k in [0, 1, 42, 2**63 + 5] for i in range(4) for z in [1, 3, 4]],
    }
    with open(os.path.join(OUT, "hashing.json"), "w") as fh:
        json.dump(hashing, fh, indent=1, sort_keys=True)

    # ---------------------------------------------------------------- apply cases
    kinds = ["sf1", "sf2", "sf3", "sf4", "sff", "cm", "cu"]
    small = SketchParams(d=3, w=16, z=3, master_seed=5)
    ops_m, keys_m = mixed_stream(14, 2000, 60, 0.3)
    ops_i = np.zeros(5000, np.uint8)
    keys_i = generate(WorkloadSpec(kind="zipf", distinct_items=300, total_ops=5000, seed=3)).keys
    for k in kinds:
        manifest[f"{k}_insert_small"] = run_case(f"{k}_insert_small", k, small, ops_i, keys_i)
        manifest[f"{k}_mixed_small"] = run_case(f"{k}_mixed_small", k, small, ops_m, keys_m)
    # uint32 keys, medium, shapes of the configs (d=4, z=4), several batches
    rng = np.random.Generator(np.random.PCG64(2017))
    distinct = np.unique(rng.integers(0, 1 << 32, size=6000, dtype=np.uint64).astype(np.uint32))[:5000]
    r = np.minimum(np.searchsorted(np.cumsum(1 / np.arange(1, 5001) / np.sum(1 / np.arange(1, 5001))),
                                   rng.random(60000), side="right"), 4999)
    ins32 = distinct[r]
    med = SketchParams(d=4, w=256, z=4, master_seed=2017)
    for k in ["sf1", "sff", "cm", "cu", "sf4"]:
        manifest[f"{k}_u32_medium"] = run_case(f"{k}_u32_medium", k, med, np.zeros(60000, np.uint8), ins32,
                                              query_keys=distinct, batches=3)
    # SFF / CM with occurrence-level interleaved deletes (cfg-3 style), u32 keys
    n_del = 12000
    victims = rng.choice(60000, size=n_del, replace=False)
    dpos = victims + (1.0 - rng.random(n_del)) * (60000 - victims)
    order = np.argsort(np.concatenate([np.arange(60000, dtype=np.float64), dpos]), kind="stable")
    ops3 = np.concatenate([np.zeros(60000, np.uint8), np.ones(n_del, np.uint8)])[order]
    keys3 = np.concatenate([ins32, ins32[victims]])[order]
    for k in ["sff", "sf4", "cm", "sf2", "sf3"]:
        manifest[f"{k}_u32_deletes"] = run_case(f"{k}_u32_deletes", k, med, ops3, keys3, query_keys=distinct)
    # non power-of-two widths (cfg-4 style: w = 12800-like modulus), u64 keys
    odd = SketchParams(d=4, w=100, w_prime=32768 + 3, master_seed=99)
    manifest["sf1_oddwidth"] = run_case("sf1_oddwidth", "sf1", odd, ops_i, keys_i)
    manifest["cm_oddwidth"] = run_case("cm_oddwidth", "cm", SketchParams(d=4, w=12800, master_seed=99), ops_i, keys_i)
    # ---------------------------------------------------------------- failures
    tiny = SketchParams(d=2, w=8, z=2, master_seed=1)
    ops_f = np.array([0, 0, 1, 0, 1, 1, 0], np.uint8)
    keys_f = np.array([5, 6, 5, 7, 6, 9, 5], np.uint64)  # delete of 9 is a phantom
    for k in ["sff", "sf4", "sf2", "sf3", "cm"]:
        manifest[f"{k}_phantom"] = run_case(f"{k}_phantom", k, tiny, ops_f, keys_f)
    manifest["sf1_unsupported"] = run_case("sf1_unsupported", "sf1", tiny, ops_f, keys_f)
    manifest["cu_unsupported"] = run_case("cu_unsupported", "cu", tiny, ops_f, keys_f)
    ops_s = np.zeros(40, np.uint8)
    keys_s = np.arange(40, dtype=np.uint64) % 7
    near = np.uint32(0xFFFFFFFF - 3)
    for k in ["sff", "sf1", "sf4"]:
        p = SketchParams(d=2, w=8, z=2, master_seed=1)
        fat_shape = (2, 8, 2) if k in ("sff", "sf4") else (2, 16)
        manifest[f"{k}_saturate"] = run_case(f"{k}_saturate", k, p, ops_s, keys_s,
                                             preset={"fat": np.full(fat_shape, near, np.uint32)})
    for k in ["cm", "cu"]:
        manifest[f"{k}_saturate"] = run_case(f"{k}_saturate", k, tiny, ops_s, keys_s,
                                             preset={"slim": np.full((2, 8), near, np.uint32)})
    with open(os.path.join(OUT, "manifest.json"), "w") as fh:
        json.dump({k: [int(a), int(b)] for k, (a, b) in manifest.items()}, fh, indent=1, sort_keys=True)
    print(json.dumps({k: [int(a), int(b)] for k, (a, b) in manifest.items()}))


if __name__ == "__main__":
    main()
