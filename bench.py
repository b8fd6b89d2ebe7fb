"""Headline benchmark: SF insert & query throughput on B200 (BASELINE.json).

One step = the SF sketch hot path over one synthetic batch:
  1. build: a fresh SFF sketch (d=4, w=65536, z=4) applies the cfg-3 stream
     (10M inserts Zipf(1.0) over 1M distinct uint32 keys + 2M occurrence-level
     deletes, 12M ops) through ``SfSketch.apply_ops`` on rank 0 (SF updates
     are order-dependent: single GPU);
  2. replicate: with N > 1 the slim is broadcast from rank 0 (NCCL/NVLink);
  3. query: the cfg-5 batch of Q point queries (default 1B uint32 keys, half
     present with Zipf(1.0) rank skew, half absent) sharded contiguously over
     the N GPUs, each answering its slice with the fused hash+gather+min kernel.
This is north_star's multi-GPU layout (strong scaling: the job is fixed, the
build stays on one GPU, the queries spread). ``--replicas`` instead runs N
independent sketches (weak scaling). Beside the headline the line reports
``insert`` and ``query`` separately (Mitems/s, fraction of the random-gather
roofline, CPU ratio), and ``cm_merge``: the cfg-2 count-min build sharded by
stream over the N GPUs and merged with one NCCL all-reduce.
value = (ops applied + queries answered) / step time (max over ranks),
Mitems/s. Inputs are device-resident for ``value``; ``e2e`` repeats the step
through the same public API from pinned HOST buffers (H2D of ops/keys and
query keys, D2H of the estimates inside the timed region).

``--impl reference`` times the reference's own CPU implementation (the
``sfsketch`` package installed unmodified in ``baseline/_ref``, numba
kernels) on the host cores for the same workload: the build single-threaded
(single-writer contract), the queries split over all host threads
(``bench.py:153-162`` of the reference), extrapolated from a bounded sample.
Without ``baseline/_ref`` it falls back to the C port of those kernels
(``oracle/``, pinned bit-exact to the reference).
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SF insert & query Mitems/s"
SEED = 2017
D, W, Z = 4, 65536, 4


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--queries", type=int, default=1_000_000_000)
    ap.add_argument("--alpha", type=float, default=1.0, help="build stream skew (cfg 3)")
    ap.add_argument("--alpha-q", type=float, default=1.0, help="query rank skew (cfg 5)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-stage-first", action="store_true",
                    help="e2e: start the staging copy before apply_ops instead of behind its upload")
    ap.add_argument("--e2e-stage", type=int, default=0,
                    help="e2e: query keys uploaded (SfSketch.stage_query_keys) before the build; 0 = none "
                         "(measured slower: the staging copy delays the build's own upload, DESIGN.md §5.1)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cm", action="store_true", help="skip the cfg-2 CM merge leg")
    ap.add_argument("--replicas", action="store_true",
                    help="N>1: one independent sketch per GPU (weak scaling) instead of the default build on rank 0 "
                         "+ slim broadcast + sharded queries")
    ap.add_argument("--shared-slim", action="store_true", help="(default; kept for old command lines)")
    ap.add_argument("--cpu-kind", default="auto", choices=["auto", "reference", "port"],
                    help="CPU baseline: the reference package in baseline/_ref (numba) or the C port")
    return ap.parse_args()


def replicas(args, world):
    return world > 1 and args.replicas


def workload_config(args, world):
    if replicas(args, world):
        par = ("replicas only: %d independent sketches, one per GPU (SF updates are order-dependent and do not "
               "shard); rank r builds its own cfg-3 stream (seed %d + r) and answers its own %d queries; no "
               "data-path collective" % (world, SEED, args.queries))
    elif world > 1:
        par = ("north_star layout: build on rank 0 (SF updates are order-dependent), NCCL broadcast of the slim, "
               "queries sharded contiguously over %d GPUs" % world)
    else:
        par = "1 GPU"
    return {
        "workload": "cfg3 SFF build (10M inserts Zipf(%.1f)/1M + 2M interleaved deletes) + cfg5 %d point queries "
                    "(50%% present Zipf(%.1f), 50%% absent) on the built slim" % (args.alpha, args.queries, args.alpha_q),
        "d": D, "w": W, "z": Z, "ops": 12_000_000, "queries": args.queries,
        "parallelism": par,
        "l2": "query keys (4 B x Q) exceed L2; L2 flushed (256 MiB write) between steps",
        "seed": SEED,
    }


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clocks + clock-event reasons sampled DURING the timed region through
    NVML (pynvml) in a background thread; nvidia-smi is the fallback."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, device_index: int, period_s: float = 0.01):
        self.idx = device_index
        self.period = period_s
        self.samples = []  # (sm_mhz, max_mhz, reason_bits)
        self.err = None
        self._stop = threading.Event()
        self.t = None

    def _handle(self):
        import pynvml
        import torch

        pynvml.nvmlInit()
        uuid = str(torch.cuda.get_device_properties(self.idx).uuid)
        try:
            return pynvml, pynvml.nvmlDeviceGetHandleByUUID("GPU-" + uuid if not uuid.startswith("GPU-") else uuid)
        except Exception:  # noqa: BLE001 - fall back to the visible-index mapping
            vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
            ids = [v for v in vis.split(",") if v.strip()]
            phys = int(ids[self.idx]) if ids and ids[self.idx].strip().isdigit() else self.idx
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(phys)

    def _run(self):
        try:
            nv, h = self._handle()
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            while not self._stop.is_set():
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((sm, mx, rs, time.perf_counter()))
                self._stop.wait(self.period)
        except Exception as e:  # noqa: BLE001
            self.err = f"nvml: {type(e).__name__}: {e}"

    def start(self):
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def stop(self, t_begin=None, t_end=None):
        self._stop.set()
        if self.t is not None:
            self.t.join(timeout=5)
        timed = [s for s in self.samples if (t_begin is None or s[3] >= t_begin) and (t_end is None or s[3] <= t_end)]
        timed = timed or self.samples
        # only samples taken under load (GpuIdle bit clear) count toward the median
        load = [s for s in timed if not (s[2] & 0x1)] or timed
        sm = [s[0] for s in load]
        reasons = sorted({nm for s in load for nm, bit in self.REASONS.items() if s[2] & bit})
        out = {"sm_mhz": statistics.median(sm) if sm else None,
               "sm_max_mhz": max(s[1] for s in self.samples) if self.samples else None,
               "reasons": reasons, "samples": len(timed), "samples_under_load": len(load),
               "source": "nvml (pynvml), 10 ms period, samples inside the timed region"}
        if self.err:
            out["error"] = self.err
        return out


def ncu_traffic(name, units):
    """DRAM bytes per launch of `name` scaled from the committed ncu --set full
    capture (profiles/ncu_traffic.json, written by tools/ncu_summary.py)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as fh:
        e = json.load(fh).get(name)
    return None if e is None else int(e["bytes_per_unit"] * units)


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    hbm, src = 6650.0, "fallback (B200_PROFILING.md)"
    if os.path.exists(p):
        with open(p) as fh:
            hbm, src = float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    gather = None
    gp = os.path.join(ROOT, "profiles", "gather_peaks.json")
    if os.path.exists(gp):
        with open(gp) as fh:
            gather = json.load(fh)
    return hbm, src, gather


# ------------------------------------------------------------------ reference arm
def ref_package():
    """The unmodified reference package installed in baseline/_ref (None if absent)."""
    p = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isfile(os.path.join(p, "sfsketch", "__init__.py")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/sfk_numba_cache")
    if p not in sys.path:
        sys.path.insert(0, p)
    try:
        import sfsketch
    except Exception:  # noqa: BLE001 - e.g. numba missing: the port stands in
        return None
    return sfsketch


def cpu_kind(args):
    if args.cpu_kind == "port":
        return "port", None
    ref = ref_package()
    if ref is None and args.cpu_kind == "reference":
        raise SystemExit("baseline/_ref holds no importable sfsketch")
    return ("reference", ref) if ref is not None else ("port", None)


def cpu_measure(args, stream, qs, threads, kind="port", ref=None):
    """The CPU path on the host: the full 12M-op cfg-3 build single-threaded
    (the reference's single-writer contract), then `qs` queries split over
    `threads` threads; kind "reference" drives the reference package's own
    SfSketch (numba; JIT warmed first as the reference's bench.py:155,181
    does), kind "port" the C restatement. Returns (value Mitems/s, build s,
    query s, sample text, sketch)."""
    from concurrent.futures import ThreadPoolExecutor

    ops = stream["ops"]
    keys64 = stream["keys"].astype(np.uint64)
    n_ops = ops.shape[0]
    if kind == "reference":
        sk = ref.SfSketch(ref.SketchParams(d=D, w=W, z=Z, master_seed=SEED), "sff")
        sk.apply_ops(ops[:1], keys64[:1])  # compile
        t0 = time.perf_counter()
        sk.apply_ops(ops[1:], keys64[1:])
        t_build = (time.perf_counter() - t0) * n_ops / (n_ops - 1)
        q64 = qs.astype(np.uint64)
        chunks = np.array_split(q64, threads)
        sk.query_many(q64[:16])  # compile
        with ThreadPoolExecutor(max_workers=threads) as pool:
            t0 = time.perf_counter()
            outs = [f.result() for f in [pool.submit(sk.query_many, c) for c in chunks]]
            t_q = time.perf_counter() - t0
        est = np.concatenate(outs)
        what = "reference sfsketch (baseline/_ref, numba)"
    else:
        from oracle import oracle as orc

        orc.lib()
        sk = orc.OracleSketch("sff", D, W, Z, None, SEED)
        t0 = time.perf_counter()
        st = sk.apply_ops(ops, keys64)
        t_build = time.perf_counter() - t0
        assert st[0] == 0
        est = np.ones(qs.shape[0], dtype=np.int64)  # pre-faulted output, as a server would reuse
        m = min(qs.shape[0], 1 << 20)
        sk.query_many(qs[:m], threads=threads, out=est[:m])  # warm
        t0 = time.perf_counter()
        sk.query_many(qs, threads=threads, out=est)
        t_q = time.perf_counter() - t0
        what = "C port of the reference kernels (oracle/)"
    t_total = t_build + t_q * (args.queries / qs.shape[0])
    value = (n_ops + args.queries) / t_total / 1e6
    sample = (f"{what}: full {n_ops:,}-op cfg-3 build on 1 thread ({t_build:.2f} s) + {qs.shape[0]:,} cfg-5 queries "
              f"on {threads} threads ({t_q:.2f} s), query time extrapolated to {args.queries:,}")
    return value, t_build, t_q, sample, sk, est


def cpu_state(kind, sk):
    """(slim, fat) of a CPU sketch of either kind, as numpy arrays."""
    if kind == "reference":
        return sk.slim.counters, sk.fat.counters
    return sk.slim, sk.fat


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_1701_04148_b200 import workloads as Wl

    kind, ref = cpu_kind(args)
    stream = Wl.cfg3(seed=SEED, alpha=args.alpha)
    sample_n = 50_000_000 if kind == "reference" else 100_000_000
    qs = Wl.query_keys(SEED + 5, stream["distinct"], args.alpha_q, 0, sample_n)
    threads = len(os.sched_getaffinity(0))
    times = []
    for k in range(args.warmup + args.steps):
        value, tb, tq, sample, _, _ = cpu_measure(args, stream, qs, threads, kind, ref)
        if k >= args.warmup:
            times.append((value, tb, tq))
    value = statistics.median([t[0] for t in times])
    tb = statistics.median([t[1] for t in times])
    tq = statistics.median([t[2] for t in times])
    n_items = 12_000_000 + args.queries
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "Mitems/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(n_items / (value * 1e6) * 1e3, 3), "higher_is_better": True,
        "scaling": "weak" if (args.gpus > 1 and args.replicas) else "strong",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic (seeded, SURVEY.md §8(d))",
        "config": workload_config(args, args.gpus),
        "cpu_baseline": {"value": round(value, 3), "unit": "Mitems/s", "cores": threads, "kind": kind,
                         "sample": sample, "cpu": cpu_model()},
        "insert": {"Mitems_s": round(12_000_000 / tb / 1e6, 3), "threads": 1},
        "query": {"Mitems_s": round(qs.shape[0] / tq / 1e6, 3), "threads": threads},
        "e2e": {"value": round(value, 3), "unit": "Mitems/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


# ------------------------------------------------------------------ CM merge leg
def run_cm_leg(args, world, rank, dev):
    """cfg 2 count-min build: every rank applies its contiguous slice of the
    10M-op stream (warp-aggregated atomics) and the replicas are summed with
    one NCCL all-reduce (distributed.sharded_cm_apply). Timed like the
    headline (CUDA events, max over ranks), not part of `value`."""
    import torch
    import torch.distributed as dist

    import paper_1701_04148_b200 as P
    from paper_1701_04148_b200 import workloads as Wl

    c = Wl.cfg2(seed=SEED)
    ops_d = torch.from_numpy(c["ops"]).to(dev)
    keys_d = torch.from_numpy(c["keys"]).to(dev)
    cm = P.CmSketch(P.SketchParams(d=D, w=W, master_seed=SEED))
    times = []
    for k in range(args.warmup + args.steps):
        cm.counters.zero_()
        cm.increment_counts.zero_()
        cm.insertions_seen = 0
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if world > 1:
            cm.sharded_apply_(ops_d, keys_d)
        else:
            cm.apply_ops(ops_d, keys_d)
        e1.record()
        torch.cuda.synchronize()
        if k >= args.warmup:
            times.append(e0.elapsed_time(e1))
    t = torch.tensor([sum(times) / len(times)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    n = int(c["ops"].shape[0])
    out = {"workload": "cfg2 CM d=4 w=65536, 10M inserts Zipf(1.0) over 1M distinct uint32 keys, stream sharded "
                       "over %d GPU(s) (global precheck, raw signed deltas, one NCCL sum all-reduce; "
                       "distributed.sharded_cm_apply)" % world if world > 1 else
                       "cfg2 CM d=4 w=65536, 10M inserts Zipf(1.0) over 1M distinct uint32 keys, 1 GPU "
                       "(CmSketch.apply_ops: device precheck + warp-aggregated atomics)",
           "ms": round(ms, 3), "Mitems_s": round(n / (ms * 1e-3) / 1e6, 2), "ops": n, "n_gpus": world}
    _, _, gather = measured_peaks()
    if gather and gather.get("red_1MiB_Gps"):
        # d atomic counter updates per op against the measured RED peak on a
        # 1 MiB L2-resident table, per GPU
        upd = n * D / (ms * 1e-3) / 1e9 / world
        out["gather"] = {"red_Gps_per_gpu": round(upd, 1), "peak_Gps": gather["red_1MiB_Gps"],
                         "frac": round(upd / gather["red_1MiB_Gps"], 4),
                         "peak_source": "profiles/gather_peaks.json (RED.ADD on a 1 MiB table)"}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        kind, ref = cpu_kind(args)
        keys64 = c["keys"].astype(np.uint64)
        if kind == "reference":
            r = ref.CmSketch(ref.SketchParams(d=D, w=W, master_seed=SEED))
            r.apply_ops(c["ops"][:1], keys64[:1])  # compile
            t0 = time.perf_counter()
            r.apply_ops(c["ops"][1:], keys64[1:])
            cpu_rate = (n - 1) / (time.perf_counter() - t0) / 1e6
            want = r.counters
        else:
            from oracle import oracle as orc

            o = orc.OracleSketch("cm", D, W, master_seed=SEED)
            t0 = time.perf_counter()
            o.apply_ops(c["ops"], keys64)
            cpu_rate = n / (time.perf_counter() - t0) / 1e6
            want = o.slim
        out["cpu_Mitems_s"] = round(cpu_rate, 2)
        out["cpu_kind"] = kind
        out["cpu_ratio"] = round(out["Mitems_s"] / cpu_rate, 1)
        assert np.array_equal(cm.counters.cpu().numpy(), want), "CM counters differ from the CPU reference"
        out["parity"] = f"counters bit-exact vs the CPU {kind}"
    return out


# ------------------------------------------------------------------ our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1701_04148_b200 as P
    from paper_1701_04148_b200 import _lib, workloads as Wl
    from paper_1701_04148_b200.sf import query_min

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # SFK_BENCH_DEVICE / SFK_BENCH_BACKEND: functional check of the N > 1 code
    # path on a one-GPU box (every rank on one device, gloo collectives); not
    # a measurement
    local_dev = int(os.environ.get("SFK_BENCH_DEVICE", local))
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    if world > 1:
        backend = os.environ.get("SFK_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    L = _lib.lib()

    rep = replicas(args, world)
    # replicas: rank r is an independent sketch over its own stream and queries
    rseed = SEED + rank if rep else SEED
    stream = Wl.cfg3(seed=rseed, alpha=args.alpha)
    n_ops = int(stream["ops"].shape[0])
    ops_d = torch.from_numpy(stream["ops"]).to(dev)
    keys_d = torch.from_numpy(stream["keys"]).to(dev)
    if rep or world == 1:
        q0, qn = 0, args.queries
    else:
        per = args.queries // world
        q0 = rank * per
        qn = per if rank < world - 1 else args.queries - q0
    gen = Wl.DeviceQueryStream(rseed + 5, stream["distinct"], args.alpha_q)
    qkeys = gen.keys(q0, qn)
    qout = torch.empty(qn, dtype=torch.int64, device=dev)
    params = P.SketchParams(d=D, w=W, z=Z, master_seed=SEED)
    sk = P.SfSketch(params, "sff")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    torch.cuda.synchronize()

    def reset():
        sk.slim.counters.zero_()
        sk.fat.counters.zero_()
        sk.slim.increment_counts.zero_()
        sk.slim.insertions_seen = 0
        sk._used_normal = False

    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]

    def step():
        ev[0].record()
        eng = 0.0
        if rank == 0 or rep:
            reset()
            sk.apply_ops(ops_d, keys_d)
            eng = float(L.sfk_engine_last_ms())
        ev[1].record()
        if world > 1 and not rep:
            sk.broadcast_slim_(src=0)
        ev[2].record()
        rc = L.sfk_min_query(sk.slim.counters.data_ptr(), sk._slim_seeds.ctypes.data, D, W, qkeys.data_ptr(),
                             _lib.KEY_U32, 0, qn, qout.data_ptr(), _lib.stream_ptr())
        _lib.check(rc, "sfk_min_query")
        ev[3].record()
        torch.cuda.synchronize()
        return [ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3]), eng]

    # nvidia-smi needs ~0.5 s to start sampling: start it before the warm-up
    clocks = ClockSampler(local_dev)
    clocks.start()
    time.sleep(1.0)
    for _ in range(args.warmup):
        step()
        flush.fill_(1)
    # correctness gate for the measured state (rank 0 vs its own last build)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = L.sfk_launch_count()
    L.sfk_engine_timing(1)
    est0 = (ctypes.c_ulonglong * 8)()
    L.sfk_engine_stats(est0, 1)
    phases = []
    t_begin = time.perf_counter()
    for _ in range(args.steps):
        phases.append(step())
        flush.fill_(1)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = L.sfk_launch_count() - launches0
    L.sfk_engine_timing(0)
    est = (ctypes.c_ulonglong * 8)()
    L.sfk_engine_stats(est, 1)
    t_end = time.perf_counter()
    clk = clocks.stop(t_begin, t_end)
    tot = np.array(phases).sum(axis=0)  # build, bcast, query, engine kernel (ms over K steps)
    step_ms_local = float(tot[:3].sum()) / args.steps
    t = torch.tensor([step_ms_local, tot[0] / args.steps, tot[1] / args.steps, tot[2] / args.steps],
                     dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    step_ms, build_ms, bcast_ms, query_ms = (float(x) for x in t.tolist())
    items = (n_ops + args.queries) * (world if rep else 1)  # whole job: every replica's ops and queries
    value = items / (step_ms * 1e-3) / 1e6

    hbm, hbm_src, gather = measured_peaks()
    # per-kernel rooflines from CUDA events on the launching stream
    q_s = float(tot[2]) / args.steps * 1e-3
    achieved_gbs = qn * 12 / q_s / 1e9
    qpath = int(L.sfk_query_last_path())
    qkern = {1: "min_query_l2 (fused key load + 4x hash + 4 L2 gathers + min + int64 store)",
             2: "min_query_smem (whole slim in one SM's shared memory)",
             3: "min_query_cluster<4,u16> (4-CTA cluster, one slim row per CTA in smem, DSMEM st.async "
                "partials, min + int64 store)",
             4: "min_query_cw<4,u16> (4-CTA cluster, one slim row per CTA in smem; warp-pipelined: per-warp "
                "512-key tiles, DSMEM st.async partials on per-warp mbarriers, packed-u16 min, coalesced int64 "
                "stores)"}.get(qpath, "?")
    rf_query = {"bound": "hbm", "achieved": round(achieved_gbs, 1), "peak": hbm, "unit": "GB/s",
                "frac": round(achieved_gbs / hbm, 4),
                "traffic": ncu_traffic({3: "query_cluster", 4: "query_cw"}.get(qpath, ""), qn), "kernel": qkern,
                "algorithmic_bytes_per_launch": int(qn * 12), "launch_ms": round(q_s * 1e3, 3),
                "peak_source": hbm_src}
    if gather:
        # the gather level the path reads from: L2 for path 1, shared memory otherwise
        key, lvl = ("gather_1MiB_Gps", "L2, 1 MiB table") if qpath == 1 else ("gather_smem128KiB_Gps", "smem")
        gpk = float(gather.get(key, 0.0))
        gachieved = qn * 4 / q_s / 1e9
        rf_query["gather"] = {"achieved_Gps": round(gachieved, 1), "peak_Gps": gpk,
                              "frac": round(gachieved / gpk, 4) if gpk else None,
                              "peak_source": f"profiles/gather_peaks.json (random 4-B loads, {lvl})"}
    rf = {"query": rf_query}
    eng_ms = float(tot[3]) / args.steps
    if rank == 0 and eng_ms > 0:
        runs = est[4] / args.steps
        # per run: its record (12 + 16 d bytes) + d slim words read and written (8 B each); 1 bit per op
        eng_bytes = runs * (12 + 16 * D + 16 * D) + n_ops / 8
        ach = eng_bytes / (eng_ms * 1e-3) / 1e9
        rf["engine"] = {"bound": "hbm", "achieved": round(ach, 2), "peak": hbm, "unit": "GB/s",
                        "frac": round(ach / hbm, 5), "traffic": ncu_traffic("engine_sff", runs),
                        "kernel": "poll_engine_k<4,2> (ordered slim engine, SFF)",
                        "algorithmic_bytes_per_launch": int(eng_bytes), "launch_ms": round(eng_ms, 3),
                        "runs_per_launch": int(runs), "peak_source": hbm_src,
                        "note": "latency-bound: runs wait on the slim cells their predecessors write; "
                                "see DESIGN.md for the critical-path depth"}
        hl = os.path.join(ROOT, "profiles", "hop_latency.json")
        if os.path.exists(hl) and args.alpha == 1.0:
            with open(hl) as fh:
                h = json.load(fh)
            floor_ms = h["cfg3_alpha1_critical_hops"] * h["hop_ns_idle"] * 1e-6
            rf["engine"]["latency_roofline"] = {
                "critical_hops": h["cfg3_alpha1_critical_hops"], "hop_ns_floor": h["hop_ns_idle"],
                "floor_ms": round(floor_ms, 3), "frac": round(floor_ms / eng_ms, 4),
                "source": "profiles/hop_latency.json (tools/hop_latency.cu ping-pong; tools/trace_engine.py hops)"}
    dominant = "engine" if "engine" in rf and eng_ms > query_ms else "query"
    roofline = dict(rf[dominant])
    roofline["dominant"] = dominant
    roofline["kernels"] = rf

    breakdown = {"build_ms": round(build_ms, 3), "bcast_ms": round(bcast_ms, 3), "query_ms": round(query_ms, 3),
                 "insert_Mitems_s": round(n_ops / (build_ms * 1e-3) / 1e6, 2) if build_ms else None,
                 "query_Mitems_s": round(args.queries / (query_ms * 1e-3) / 1e6, 2) if query_ms else None}

    # ------------------------------------------------ e2e through the API from host buffers
    e2e = None
    if not args.no_e2e:
        ops_h = torch.from_numpy(stream["ops"]).pin_memory()
        keys_h = torch.from_numpy(stream["keys"]).pin_memory()
        qk_h = torch.empty(qn, dtype=torch.uint32).pin_memory()
        qk_h.copy_(qkeys)
        qo_h = torch.empty(qn, dtype=torch.int64).pin_memory()
        e_times, e_split = [], []
        for k in range(args.warmup + args.steps):
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            # optionally, the first query keys upload on a side stream before the build
            staged = (sk.stage_query_keys(qk_h, args.e2e_stage, with_next_apply=not args.e2e_stage_first)
                      if args.e2e_stage > 0 else None)
            if rank == 0 or rep:
                reset()
                sk.apply_ops(ops_h, keys_h)  # H2D inside the API call
            if world > 1 and not rep:
                sk.broadcast_slim_(src=0)
            t1 = time.perf_counter()
            sk.query_many_host(qk_h, out=qo_h, staged=staged)  # host keys in, host int64 estimates out
            del staged
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            e = t2 - t0
            if k >= args.warmup:
                e_times.append(e)
                e_split.append((t1 - t0, t2 - t1))
            flush.fill_(1)
        et = torch.tensor([sum(e_times) / len(e_times)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        wire = int(L.sfk_host_query_config(_lib.HQ_LAST_WIRE, -1))
        wb = {_lib.WIRE_C16: 2, _lib.WIRE_U32: 4}.get(wire, 8)
        sc = sk.slim.counters.to(torch.int64)
        dict_bytes = int(torch.unique(sc[sc >= 0xF800]).numel()) * 4 if wire == _lib.WIRE_C16 else 0
        # per step: the apply's ops + keys and its 24-B result; the query keys,
        # the wire dictionary's set (16 KiB + flag) back and the sorted
        # dictionary out, and the narrowed estimates
        e2e = {"value": round(items / float(et.item()) / 1e6, 3), "unit": "Mitems/s",
               "h2d_bytes_per_step": int((n_ops * 5 if (rank == 0 or rep) else 0) + qn * 4 + dict_bytes),
               "d2h_bytes_per_step": int(qn * wb + (16388 if wire != _lib.WIRE_I64 else 0) + 24),
               "wire": {_lib.WIRE_C16: "u16 codes", _lib.WIRE_U32: "u32", _lib.WIRE_I64: "int64"}.get(wire, "?"),
               "apply_ms": round(sum(a for a, _ in e_split) / len(e_split) * 1e3, 3),
               "query_ms": round(sum(b for _, b in e_split) / len(e_split) * 1e3, 3),
               "staged_query_keys": int(min(args.e2e_stage, qn)) if args.e2e_stage > 0 else 0,
               "note": "apply_ops from pinned host ops/keys (staged_query_keys > 0: that many query keys upload "
                       "on a side stream from before the build, SfSketch.stage_query_keys); queries through "
                       "SfSketch.query_many_host "
                       "(sfk_min_query_host: chunked H2D -> query kernel -> narrowed D2H, host threads widen "
                       "into the int64 output); wall clock, max over ranks"}
        # the estimates must equal the device-resident run's
        assert torch.equal(qo_h.to(dev), qout), "e2e estimates differ from device-resident run"

    # ------------------------------------------------ CM merge leg (cfg 2), reported beside the headline
    cm_leg = None if args.no_cm else run_cm_leg(args, world, rank, dev)

    # ------------------------------------------------ parity gate + CPU baseline (rank 0, N=1)
    cpu = cpu_port = None
    cpu_build_s = cpu_q_rate = None
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        kind, ref = cpu_kind(args)
        threads = len(os.sched_getaffinity(0))
        sample_n = 50_000_000
        qs = qkeys[:sample_n].cpu().numpy()
        gpu_slim, gpu_fat = sk.slim.counters.cpu().numpy(), sk.fat.counters.cpu().numpy()
        gpu_est = qout[:sample_n].cpu().numpy()
        for k in ([kind, "port"] if kind == "reference" else ["port"]):
            v, tb, tq, sample, csk, est_c = cpu_measure(args, stream, qs, threads, k, ref)
            c_slim, c_fat = cpu_state(k, csk)
            ok = (np.array_equal(gpu_slim, c_slim) and np.array_equal(gpu_fat, c_fat)
                  and np.array_equal(gpu_est, est_c))
            assert ok, f"GPU state differs from the CPU {k}"
            entry = {"value": round(v, 3), "unit": "Mitems/s", "cores": threads, "kind": k, "sample": sample,
                     "build_s": round(tb, 3), "query_Mitems_s": round(qs.shape[0] / tq / 1e6, 2),
                     "parity": "slim, fat and the sample's estimates bit-exact vs the GPU run", "cpu": cpu_model()}
            if cpu is None:
                cpu, cpu_build_s, cpu_q_rate = entry, tb, qs.shape[0] / tq / 1e6
            else:
                cpu_port = entry

    # ------------------------------------------------ insert and query as first-class figures
    g4 = float(gather.get("gather_4MiB_Gps", 0.0)) if gather else 0.0
    ins_rate = n_ops * (world if rep else 1) / (build_ms * 1e-3) / 1e6 if build_ms else None
    insert = {"Mitems_s": round(ins_rate, 2) if ins_rate else None, "ms": round(build_ms, 3), "ops": n_ops,
              "engine_ms": round(eng_ms, 3) if eng_ms > 0 else None, "touches_per_item": 8,
              "touches_note": "SURVEY §8(d): 4 fat RMW + 4 slim reads per insert (+ the slim raises), "
                              "SFF deletes 4 fat RMW + 4 bucket reads + 4 slim RMW"}
    if ins_rate and g4:
        insert["gather"] = {"achieved_Gps": round(ins_rate * 8 / 1e3, 2), "peak_Gps": g4,
                            "frac": round(ins_rate * 8 / 1e3 / g4, 4),
                            "peak_source": "profiles/gather_peaks.json (random 4-B loads, 4 MiB L2-resident table)"}
    if "engine" in rf and "latency_roofline" in rf["engine"]:
        insert["latency_roofline"] = rf["engine"]["latency_roofline"]
    if cpu_build_s:
        insert["cpu_Mitems_s"] = round(n_ops / cpu_build_s / 1e6, 2)
        insert["cpu_threads"] = 1
        insert["cpu_ratio"] = round(ins_rate / insert["cpu_Mitems_s"], 1)
    q_rate = args.queries * (world if rep else 1) / (query_ms * 1e-3) / 1e6 if query_ms else None
    query = {"Mitems_s": round(q_rate, 1) if q_rate else None, "ms": round(query_ms, 3), "queries": args.queries,
             "n_gpus": world, "per_gpu_Mitems_s": round(qn / q_s / 1e6, 1),
             "kernel": qkern, "touches_per_item": 4, "hbm_frac": rf_query["frac"]}
    if "gather" in rf_query:
        query["gather"] = rf_query["gather"]
    if cpu_q_rate:
        query["cpu_Mitems_s"] = round(cpu_q_rate, 1)
        query["cpu_threads"] = len(os.sched_getaffinity(0))
        query["cpu_ratio"] = round(q_rate / cpu_q_rate, 1)
    if world > 1 and not rep:
        query["bcast_ms"] = round(bcast_ms, 3)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "Mitems/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(step_ms, 3), "higher_is_better": True,
            "scaling": "weak" if (rep or world == 1) else "strong",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic (seeded, SURVEY.md §8(d))",
            "config": workload_config(args, world), "insert": insert, "query": query, "breakdown": breakdown,
            "roofline": roofline, "cpu_baseline": cpu, "cpu_baseline_port": cpu_port, "e2e": e2e,
            "cm_merge": cm_leg, "gpu_launches": int(launches),
            "gpu_launches_note": "own kernels only (sfk_launch_count); CUB radix-sort/scan launches not counted",
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
