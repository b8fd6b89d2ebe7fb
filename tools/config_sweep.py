"""All five BASELINE.json configurations on one GPU: build (insert/delete)
and query throughput through the public API, each checked bit-exact against
the CPU oracle (test infrastructure), with the rate also expressed as a
fraction of the measured random-gather roofline (profiles/gather_peaks.json).

Usage: python tools/config_sweep.py [cfg ...]   (cfg in 1 2 3 4 5 v b; default 1-5;
       v = SF2/SF3/SF4 on the cfg-3 stream; b = Count / CML on the cfg-2
       stream and the oracle-assisted slim on the cfg-3 inserts)
Prints one JSON line per measurement; profiles/<round>/config_sweep.jsonl
keeps the committed copy."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1701_04148_b200 as P  # noqa: E402
from paper_1701_04148_b200 import _lib, workloads as W  # noqa: E402
from oracle import oracle as orc  # noqa: E402  (checker only)

GP = json.load(open(os.path.join(ROOT, "profiles", "gather_peaks.json")))
REPS = 3
dev = torch.device("cuda", 0)
L = _lib.lib()


def timed(fn, reps=REPS):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def emit(**kw):
    print(json.dumps(kw), flush=True)


def gather_frac(items_per_s, touches, peak_key):
    pk = GP[peak_key] * 1e9
    return round(items_per_s * touches / pk, 4)


def build_case(name, kind, params, ops, keys, keys_u64, touches, peak_key, qkeys=None, qkeys_u64=None):
    ops_d = torch.from_numpy(ops).to(dev)
    keys_d = torch.from_numpy(keys).to(dev)
    holder = {}

    def mk():
        if kind == "cm":
            return P.CmSketch(params)
        if kind == "cu":
            return P.CuSketch(params)
        return P.SfSketch(params, kind)

    def run():
        holder["sk"] = mk()
        holder["sk"].apply_ops(ops_d, keys_d)

    run()  # warm
    ms = timed(run)
    sk = holder["sk"]
    o = orc.OracleSketch(kind, params.d, params.w, params.z, params.w_prime if kind in ("sf1", "sf2", "sf3") else None,
                         params.master_seed)
    t0 = time.perf_counter()
    st = o.apply_ops(ops, keys_u64)
    cpu_s = time.perf_counter() - t0
    cnt = sk.slim.counters if isinstance(sk, P.SfSketch) else sk.counters
    ok = st[0] == 0 and np.array_equal(cnt.cpu().numpy(), o.slim)
    if isinstance(sk, P.SfSketch):
        ok = ok and np.array_equal(sk.fat.counters.cpu().numpy(), o.fat)
    n = int(ops.shape[0])
    rate = n / (ms * 1e-3)
    emit(cfg=name, op="build", kind=kind, ops=n, ms=round(ms, 3), Mitems_s=round(rate / 1e6, 2),
         gather_roofline={"touches_per_item": touches, "peak": peak_key, "frac": gather_frac(rate, touches, peak_key)},
         cpu_port_1thread_Mitems_s=round(n / cpu_s / 1e6, 2), bit_exact_vs_oracle=bool(ok))
    if qkeys is not None:
        qd = torch.from_numpy(qkeys).to(dev)
        out = {}

        def q():
            out["e"] = sk.query_many(qd)

        q()
        qms = timed(q)
        ok_q = np.array_equal(out["e"].cpu().numpy(), o.query_many(qkeys_u64, threads=orc.max_threads()))
        nq = int(qkeys.shape[0])
        qrate = nq / (qms * 1e-3)
        emit(cfg=name, op="query", kind=kind, queries=nq, ms=round(qms, 3), Mitems_s=round(qrate / 1e6, 2),
             path={1: "l2", 2: "smem", 3: "cluster"}.get(int(L.sfk_query_last_path())),
             gather_roofline={"touches_per_item": params.d, "peak": peak_key,
                              "frac": gather_frac(qrate, params.d, peak_key)},
             bit_exact_vs_oracle=bool(ok_q))
    return sk


def cfg1():
    c = W.cfg1(seed=2017)
    build_case("cfg1", "sf1", P.SketchParams(d=4, w=16384, w_prime=65536, master_seed=2017), c["ops"], c["keys"],
               c["keys"].astype(np.uint64), 8, "gather_1MiB_Gps", c["distinct"], c["distinct"].astype(np.uint64))


def cfg2():
    c = W.cfg2(seed=2017)
    p = P.SketchParams(d=4, w=65536, master_seed=2017)
    build_case("cfg2", "cm", p, c["ops"], c["keys"], c["keys"].astype(np.uint64), 4, "red_1MiB_Gps")
    build_case("cfg2", "cu", p, c["ops"], c["keys"], c["keys"].astype(np.uint64), 8, "gather_1MiB_Gps")


def cfg3():
    for a in (0.5, 1.0, 1.5):
        c = W.cfg3(seed=2017, alpha=a)
        build_case(f"cfg3 alpha={a}", "sff", P.SketchParams(d=4, w=65536, z=4, master_seed=2017), c["ops"], c["keys"],
                   c["keys"].astype(np.uint64), 8, "gather_4MiB_Gps", c["distinct"], c["distinct"].astype(np.uint64))


def variants():
    """SF2 / SF3 / SF4 on the cfg-3 stream (alpha = 1.0):
    not a BASELINE config, reported beside it."""
    c = W.cfg3(seed=2017, alpha=1.0)
    for v, wp in (("sf2", 262144), ("sf3", 262144), ("sf4", None)):
        build_case("cfg3-stream " + v, v, P.SketchParams(d=4, w=65536, z=4, w_prime=wp, master_seed=2017), c["ops"],
                   c["keys"], c["keys"].astype(np.uint64), 8, "gather_4MiB_Gps", c["distinct"],
                   c["distinct"].astype(np.uint64))


def cfg4():
    c = W.cfg4(seed=2017)
    recs = c["records"]
    q = c["distinct"][:10_000_000]
    build_case("cfg4", "sf1", P.SketchParams(d=4, w=12800, w_prime=4194304, master_seed=2017), c["ops"], recs,
               orc.keys_from_records(recs), 8, "gather_64MiB_Gps", q, orc.keys_from_records(q))


def cfg5():
    c = W.cfg3(seed=2017, alpha=1.0)
    sk = P.SfSketch(P.SketchParams(d=4, w=65536, z=4, master_seed=2017), "sff")
    sk.apply_ops(torch.from_numpy(c["ops"]).to(dev), torch.from_numpy(c["keys"]).to(dev))
    nq = 1_000_000_000
    keys = torch.empty(nq, dtype=torch.uint32, device=dev)
    out = {}
    slim_h = sk.slim.counters.cpu().numpy()
    for aq in (0.0, 0.5, 1.0, 1.5, 2.0, 2.5, 3.0):
        W.DeviceQueryStream(2017 + 5, c["distinct"], aq).keys(0, nq, out=keys)

        def q():
            out["e"] = sk.query_many(keys)

        q()
        ms = timed(q)
        s = keys[:2_000_000].cpu().numpy().astype(np.uint64)
        ok = np.array_equal(out["e"][:2_000_000].cpu().numpy(),
                            orc.min_query(slim_h, sk._slim_seeds, s, threads=orc.max_threads()))
        rate = nq / (ms * 1e-3)
        emit(cfg="cfg5", op="query", alpha_q=aq, queries=nq, ms=round(ms, 3), Mitems_s=round(rate / 1e6, 2),
             path={1: "l2", 2: "smem", 3: "cluster"}.get(int(L.sfk_query_last_path())),
             hbm_GBps_12B=round(nq * 12 / (ms * 1e-3) / 1e9, 1),
             gather_roofline={"touches_per_item": 4, "peak": "gather_smem128KiB_Gps",
                              "frac": gather_frac(rate, 4, "gather_smem128KiB_Gps")},
             bit_exact_sample_2M_vs_oracle=bool(ok))
        out.clear()


def baselines():
    """Count / CML on the cfg-2 stream (Count with
    cfg-3-style deletes) and the oracle-assisted slim (rank 3) on the cfg-3
    inserts with their exact post-insert counts: not BASELINE configs."""
    p = P.SketchParams(d=4, w=65536, z=4, master_seed=2017)
    seeds = P.hashing.seed_array(2017, 0, 4)
    c2 = W.cfg2(seed=2017)
    c3 = W.cfg3(seed=2017, alpha=1.0)
    q = c2["distinct"][:1_000_000]
    qd = torch.from_numpy(q).to(dev)
    cases = [
        ("count", c3["ops"], c3["keys"]),
        ("cml", np.zeros(c2["keys"].size, np.uint8), c2["keys"]),
    ]
    for kind, ops, keys in cases:
        ops_d, keys_d = torch.from_numpy(ops).to(dev), torch.from_numpy(keys).to(dev)
        holder = {}

        def run():
            holder["sk"] = P.CountSketch(p) if kind == "count" else P.CmlSketch(p)
            holder["sk"].apply_ops(ops_d, keys_d)

        run()
        ms = timed(run)
        sk = holder["sk"]
        t0 = time.perf_counter()
        if kind == "count":
            ref = np.zeros((4, 65536), np.int32)
            st = orc.count_apply(ref, seeds, ops, keys.astype(np.uint64))
            ok = np.array_equal(sk.counters.cpu().numpy(), ref)
        else:
            ref = np.zeros((4, 65536), np.uint16)
            st = orc.cml_apply(ref, seeds, ops, keys.astype(np.uint64), 1.08, 2017, 0)
            ok = np.array_equal(sk.exponents.cpu().numpy(), ref)
        cpu_s = time.perf_counter() - t0
        n = int(ops.size)
        emit(cfg="cfg2-stream" if kind == "cml" else "cfg3-stream", op="build", kind=kind, ops=n, ms=round(ms, 3),
             Mitems_s=round(n / (ms * 1e-3) / 1e6, 2), cpu_port_1thread_Mitems_s=round(n / cpu_s / 1e6, 2),
             bit_exact_vs_oracle=bool(ok and st[0] == 0))
        out = {}

        def qq():
            out["e"] = sk.query_many(qd)

        qq()
        qms = timed(qq)
        if kind == "count":
            want = orc.count_query(ref, seeds, q.astype(np.uint64))
        else:
            want = orc.cml_value(orc.cml_min_exp(ref, seeds, q.astype(np.uint64)), 1.08)
        emit(cfg="cfg2-distinct", op="query", kind=kind, queries=int(q.size), ms=round(qms, 3),
             Mitems_s=round(q.size / (qms * 1e-3) / 1e6, 2),
             bit_exact_vs_oracle=bool(np.array_equal(out["e"].cpu().numpy(), want)))
    # oracle-assisted: the cfg-3 inserts with exact running counts
    keys = c3["keys"][c3["ops"] == 0]
    _, inv = np.unique(keys, return_inverse=True)
    order = np.argsort(inv, kind="stable")
    s_ = inv[order]
    head = np.concatenate([[True], s_[1:] != s_[:-1]])
    starts = np.where(head)[0]
    tc = np.empty(keys.size, np.int64)
    tc[order] = np.arange(keys.size) - np.repeat(starts, np.diff(np.append(starts, keys.size))) + 1
    keys_d, tc_d = torch.from_numpy(keys).to(dev), torch.from_numpy(tc).to(dev)
    holder = {}

    def orun():
        holder["sk"] = P.SfSketch(p, "sff")
        holder["sk"].oracle_assisted_apply(keys_d, tc_d)

    orun()
    ms = timed(orun)
    ref = np.zeros((4, 65536), np.uint32)
    inc = np.zeros(4, np.int64)
    t0 = time.perf_counter()
    st = orc.oracle_slim_apply(ref, seeds, keys.astype(np.uint64), tc, inc)
    cpu_s = time.perf_counter() - t0
    ok = st[0] == 0 and np.array_equal(holder["sk"].slim.counters.cpu().numpy(), ref)
    emit(cfg="cfg3-inserts", op="oracle_assisted_apply", ops=int(keys.size), ms=round(ms, 3),
         Mitems_s=round(keys.size / (ms * 1e-3) / 1e6, 2),
         cpu_port_1thread_Mitems_s=round(keys.size / cpu_s / 1e6, 2), bit_exact_vs_oracle=bool(ok))


if __name__ == "__main__":
    which = sys.argv[1:] or ["1", "2", "3", "4", "5"]
    for w_ in which:
        {"1": cfg1, "2": cfg2, "3": cfg3, "4": cfg4, "5": cfg5, "v": variants, "b": baselines}[w_]()
        torch.cuda.empty_cache()
