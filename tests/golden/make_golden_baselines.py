"""Regenerate the Count / CML / oracle-assisted golden fixtures by running the
REFERENCE implementation (build container only: it imports /root/reference):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_baselines.py

Writes tests/golden/baselines/*.npz. Each fixture holds the inputs (params,
ops, keys, preset state, CML base / rng seed, oracle true counts, batch
split) and the reference's outputs (counters or exponents, insertions_seen,
status / op index, query answers, the export payload and the collector's
answers for it).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from sfsketch import CmlSketch, CountSketch, SfSketch, SketchParams, export_slim, import_slim  # noqa: E402
from sfsketch.workloads import WorkloadSpec, generate  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "baselines")
STATUS = {"PhantomDeletionError": 1, "SaturationError": 2, "UnsupportedOperationError": 3}


def apply(sk, ops, keys, batches):
    bounds = np.linspace(0, len(ops), batches + 1).astype(int)
    for a, b in zip(bounds[:-1], bounds[1:]):
        try:
            sk.apply_ops(ops[a:b], keys[a:b])
        except Exception as e:  # noqa: BLE001 - the reference's status exceptions
            return STATUS[type(e).__name__], a + int(str(e).split(":")[0].split()[1])
    return 0, -1


def common(kind, params, ops, keys, batches, status, op_index, q_keys, q, payload):
    col = import_slim(payload)
    return {"kind": np.array(kind), "d": np.int64(params.d), "w": np.int64(params.w),
            "master_seed": np.uint64(params.master_seed), "ops": np.ascontiguousarray(ops, dtype=np.uint8),
            "keys": np.ascontiguousarray(keys), "batches": np.int64(batches), "status": np.int64(status),
            "op_index": np.int64(op_index), "query_keys": np.ascontiguousarray(q_keys), "query": q,
            "export": np.frombuffer(payload, dtype=np.uint8), "collector_query": col.query_many(q_keys)}


def count_case(name, params, ops, keys, batches=1, preset=None, q_keys=None):
    sk = CountSketch(params)
    if preset is not None:
        sk.counters[...] = preset
    pre = sk.counters.copy()
    status, idx = apply(sk, ops, keys, batches)
    q_keys = np.unique(keys)[:4096] if q_keys is None else q_keys
    fx = common("count", params, ops, keys, batches, status, idx, q_keys, sk.query_many(q_keys), export_slim(sk))
    fx.update({"pre_counters": pre, "counters": sk.counters.copy(), "seen": np.int64(sk.insertions_seen)})
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **fx)
    return status, idx


def cml_case(name, params, ops, keys, batches=1, base=1.08, rng_seed=None, preset=None, q_keys=None):
    sk = CmlSketch(params, base=base, rng_seed=rng_seed)
    if preset is not None:
        sk.exponents[...] = preset
    pre = sk.exponents.copy()
    status, idx = apply(sk, ops, keys, batches)
    q_keys = np.unique(keys)[:4096] if q_keys is None else q_keys
    payload = export_slim(sk)
    fx = common("cml", params, ops, keys, batches, status, idx, q_keys, sk.query_many(q_keys), payload)
    col = import_slim(payload, cml_base=base)
    fx.update({"pre_exponents": pre, "exponents": sk.exponents.copy(), "seen": np.int64(sk.insertions_seen),
               "base": np.float64(base), "rng_seed": np.uint64(sk.rng_seed),
               "collector_query": col.query_many(q_keys)})
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **fx)
    return status, idx


def oracle_case(name, params, keys, true_counts, batches=1, preset=None, q_keys=None):
    sk = SfSketch(params, "sff")
    if preset is not None:
        sk.slim.counters[...] = preset
    pre = sk.slim.counters.copy()
    bounds = np.linspace(0, len(keys), batches + 1).astype(int)
    status, idx = 0, -1
    for a, b in zip(bounds[:-1], bounds[1:]):
        try:
            sk.oracle_assisted_apply(keys[a:b], true_counts[a:b])
        except Exception as e:  # noqa: BLE001
            status, idx = STATUS[type(e).__name__], a + int(str(e).split(":")[0].split()[1])
            break
    q_keys = np.unique(keys)[:4096] if q_keys is None else q_keys
    fx = {"kind": np.array("oracle"), "d": np.int64(params.d), "w": np.int64(params.w),
          "master_seed": np.uint64(params.master_seed), "keys": np.ascontiguousarray(keys),
          "true_counts": np.ascontiguousarray(true_counts, dtype=np.int64), "batches": np.int64(batches),
          "status": np.int64(status), "op_index": np.int64(idx), "pre_slim": pre,
          "slim": sk.slim.counters.copy(), "inc": sk.slim.increment_counts.copy(),
          "seen": np.int64(sk.slim.insertions_seen), "query_keys": np.ascontiguousarray(q_keys),
          "query": sk.query_many(q_keys)}
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **fx)
    return status, idx


def main():
    os.makedirs(OUT, exist_ok=True)
    man = {}
    wl = generate(WorkloadSpec(kind="zipf", distinct_items=80, total_ops=3000, zipf_skew=1.0, seed=21,
                               deletion_mode="interleaved", delete_prob=0.3))
    ops_m, keys_m = wl.ops, wl.keys
    keys_i = generate(WorkloadSpec(kind="zipf", distinct_items=400, total_ops=6000, seed=8)).keys
    ops_i = np.zeros(keys_i.shape[0], np.uint8)
    rng = np.random.Generator(np.random.PCG64(1701))
    distinct = np.unique(rng.integers(0, 1 << 32, size=7000, dtype=np.uint64).astype(np.uint32))[:5000]
    r = np.minimum(np.searchsorted(np.cumsum(1 / np.arange(1, 5001) / np.sum(1 / np.arange(1, 5001))),
                                   rng.random(50000), side="right"), 4999)
    ins32 = distinct[r]
    # ------------------------------------------------------------ Count
    for d in (3, 4, 5):
        p = SketchParams(d=d, w=16, master_seed=5 + d)
        man[f"count_mixed_d{d}"] = count_case(f"count_mixed_d{d}", p, ops_m, keys_m)
        man[f"count_insert_d{d}"] = count_case(f"count_insert_d{d}", p, ops_i, keys_i)
    med = SketchParams(d=4, w=256, master_seed=2017)
    man["count_u32_medium"] = count_case("count_u32_medium", med, np.zeros(ins32.size, np.uint8), ins32,
                                         batches=3, q_keys=distinct)
    tiny = SketchParams(d=2, w=8, master_seed=1)
    ops_s = np.array([0, 1, 0, 0, 1, 0, 0, 0, 1, 1, 0, 0] * 3, np.uint8)
    keys_s = (np.arange(ops_s.size, dtype=np.uint64) * 7) % 5
    man["count_sat_hi"] = count_case("count_sat_hi", tiny, ops_s, keys_s,
                                     preset=np.full((2, 8), 2147483647 - 2, np.int32))
    man["count_sat_lo"] = count_case("count_sat_lo", tiny, ops_s, keys_s,
                                     preset=np.full((2, 8), -2147483648 + 2, np.int32))
    man["count_preset_signed"] = count_case(
        "count_preset_signed", SketchParams(d=4, w=8, master_seed=3), ops_m[:500], keys_m[:500],
        preset=rng.integers(-50, 50, size=(4, 8)).astype(np.int32))
    # ------------------------------------------------------------ CML
    small = SketchParams(d=3, w=16, master_seed=5)
    man["cml_insert_small"] = cml_case("cml_insert_small", small, ops_i, keys_i)
    man["cml_insert_base2"] = cml_case("cml_insert_base2", small, ops_i, keys_i, base=2.0, rng_seed=99)
    man["cml_u32_medium"] = cml_case("cml_u32_medium", SketchParams(d=4, w=256, master_seed=2017),
                                     np.zeros(ins32.size, np.uint8), ins32, batches=4, q_keys=distinct)
    man["cml_u32_base101"] = cml_case("cml_u32_base101", SketchParams(d=4, w=64, master_seed=7),
                                      np.zeros(ins32.size, np.uint8), ins32, batches=2, base=1.01)
    man["cml_unsupported"] = cml_case("cml_unsupported", small, ops_m[:400], keys_m[:400])
    man["cml_saturate"] = cml_case("cml_saturate", SketchParams(d=2, w=8, master_seed=1), np.zeros(60, np.uint8),
                                   np.arange(60, dtype=np.uint64) % 5, base=1.000001,
                                   preset=np.full((2, 8), 0xFFFF - 2, np.uint16))
    # ------------------------------------------------------------ oracle-assisted (SfSketch)
    keys_o = ins32[:20000]
    _, inv = np.unique(keys_o, return_inverse=True)
    cnt = np.zeros(inv.max() + 1, np.int64)
    tc = np.empty(keys_o.size, np.int64)
    for t, k in enumerate(inv):
        cnt[k] += 1
        tc[t] = cnt[k]
    man["oracle_true_counts"] = oracle_case("oracle_true_counts", SketchParams(d=4, w=128, z=4, master_seed=2017),
                                            keys_o, tc, batches=3, q_keys=distinct)
    noisy = tc + rng.integers(-3, 4, size=tc.size)
    man["oracle_noisy_counts"] = oracle_case("oracle_noisy_counts", SketchParams(d=3, w=50, z=4, master_seed=9),
                                             keys_o, noisy, q_keys=distinct)
    big = np.full(40, 1 << 40, np.int64)
    man["oracle_saturate"] = oracle_case("oracle_saturate", SketchParams(d=2, w=8, z=2, master_seed=1),
                                         np.arange(40, dtype=np.uint64) % 6, big,
                                         preset=np.full((2, 8), 0xFFFFFFFF - 3, np.uint32))
    with open(os.path.join(OUT, "manifest.json"), "w") as fh:
        json.dump({k: [int(a), int(b)] for k, (a, b) in man.items()}, fh, indent=1, sort_keys=True)
    print(json.dumps({k: [int(a), int(b)] for k, (a, b) in man.items()}))


if __name__ == "__main__":
    main()
