// Parallel, bit-exact batch update engine for the SF sketch (SF1, SFF), the
// CU baseline and the exact-validation path of the CM baseline.
//
// The reference applies ops one at a time (_kernels.py:244-384, 62-115).
// This file computes the same final state with a fixed pipeline of
// data-parallel passes:
//
//   1. hash_emit     fused key load + hash: for every op t and row i emit the
//                    counter cell it touches as a (cell, t|op|slot) pair.
//   2. radix sort    stable by cell (CUB onesweep), so every cell's ops sit
//                    contiguously in stream order.
//   3. segscan       a segmented prefix scan over the sorted pairs. Fat
//                    counts commute, so the fat value right after op t is
//                    initial + (#inserts - #deletes at that cell up to t):
//                    per-op observations (post-insert own count -> b_min,
//                    bucket max after a delete -> clamp), exact
//                    saturation/phantom detection (first failing op t* =
//                    atomicMin), the final fat, and for the slim cells each
//                    op's rank in its cell and its predecessor op.
//   4. runs_mark     consecutive same-key ops whose d slim cells were last
//                    touched by that same key form a "run"; a run is
//                    contiguous in the row-0 sorted order and is replayed
//                    by one thread in registers.
//   5. slim_engine   ordered dataflow engine over runs: each slim cell is a
//                    64-bit word (seq << 32 | value); a run whose head has
//                    rank r_i in cell i waits until seq_i == r_i for all its
//                    cells, replays its ops, and publishes (r_i + L, value)
//                    with one store per cell. Runs are claimed in stream
//                    order of their heads, so the earliest unfinished run is
//                    always ready and the engine cannot deadlock.
//
// Insert-only runs collapse in closed form (b_min strictly increases along
// a same-key insert run, so once a raise happens every later op raises):
// s raises give c_i' = max(c_i, m0 + s).
#include <cstring>
#include <cub/cub.cuh>

#include "sfk_common.cuh"

namespace sfk {

constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;
constexpr int ENGINE_BLOCKS_PER_SM = 1;
// default replay budget: a long run never stalls the other lanes of its warp
// for more than ~this many ops
constexpr uint32_t REPLAY_BUDGET = 1024;
// SFF runs with deletes of at most this many ops replay op by op (uniform code)
#ifndef SFK_SHORT_RUN_MAX
#define SFK_SHORT_RUN_MAX 32
#endif
constexpr bool SHORT_RUNS = SFK_SHORT_RUN_MAX > 0;
constexpr uint32_t SHORT_RUN_MAX = SFK_SHORT_RUN_MAX;
// runs with per-op caps (SF2, CML, oracle-assisted) of at most this many ops
// replay from caps loaded into registers when the run is claimed
constexpr int SHORT_CAPS = 8;
// engine run claiming: run ids per warp atomic, and how far ahead of a claim
// the run records are prefetched into L2
// poll-loop backoff: a warp that made no progress for SFK_IDLE_SPINS
// iterations sleeps up to SFK_IDLE_MAX_NS (0: never sleeps)
// engine lanes per SM: threads of its one block per SM (warp multiple)
// link records are written once and read back in other passes: streaming
// (evict-first) stores keep them from displacing the scans' working sets in L2
#ifndef SFK_LINKS_STREAMING
#define SFK_LINKS_STREAMING 1
#endif
#ifndef SFK_RUNREC_ALIGN
#define SFK_RUNREC_ALIGN alignas(32)
#endif
#ifndef SFK_ENGINE_THREADS
#define SFK_ENGINE_THREADS 256
#endif
#ifndef SFK_IDLE_SPINS
#define SFK_IDLE_SPINS 4
#endif
#ifndef SFK_IDLE_MAX_NS
#define SFK_IDLE_MAX_NS 0
#endif
#ifndef SFK_CLAIM_POOL
#define SFK_CLAIM_POOL 64
#endif
#ifndef SFK_CLAIM_PREFETCH
#define SFK_CLAIM_PREFETCH 16384
#endif
constexpr uint32_t CLAIM_POOL = SFK_CLAIM_POOL;
constexpr uint32_t CLAIM_PREFETCH = SFK_CLAIM_PREFETCH;

static uint32_t engine_budget() {
  static int v = -1;
  if (v < 0) {
    const char* s = getenv("SFK_ENGINE_BUDGET");  // tuning knob
    v = s ? atoi(s) : (int)REPLAY_BUDGET;
    if (v < 32) v = (int)REPLAY_BUDGET;
  }
  return (uint32_t)v;
}

static int engine_blocks_per_sm() {
  static int v = -1;
  if (v < 0) {
    const char* s = getenv("SFK_ENGINE_BLOCKS_PER_SM");  // tuning knob
    v = s ? atoi(s) : ENGINE_BLOCKS_PER_SM;
    if (v < 1 || v > 8) v = ENGINE_BLOCKS_PER_SM;
  }
  return v;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---------------------------------------------------------------- shared state
struct Ctl {
  uint32_t fail_t;           // first failing op (NONE32 if none)
  uint32_t n_runs;           // runs of the slim engine
  unsigned long long n_ins;  // inserts applied (t < t*)
  uint32_t qhead, qtail;     // engine ready queue
  uint32_t executed;         // engine runs finished
  uint32_t bad_op;           // first op whose code is not 0 / 1 (NONE32: none); the batch is then a no-op
};

// One 32-B sector in a single 256-bit store (STG.E.256 on sm_100): the
// scattered link / run records are whole sectors, and one store request per
// sector instead of two halves the L2 store requests.
__device__ __forceinline__ void st_sector(void* p, const uint4& a, const uint4& b) {
#if SFK_LINKS_STREAMING
  asm volatile("st.global.cs.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(a.x), "r"(a.y), "r"(a.z),
               "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
               : "memory");
#else
  asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(a.x), "r"(a.y), "r"(a.z),
               "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
               : "memory");
#endif
}

// and one 256-bit read-only load of a whole 32-B record
__device__ __forceinline__ void ld_sector(const void* p, uint4& a, uint4& b) {
  asm volatile("ld.global.nc.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
               : "l"(p));
}

// ---------------------------------------------------------------- 1. hash_emit
// kind: 0 bucketed (SFF/SF4: cell = bucket, slot in the low bits of val)
//       1 flat fat (cell = fat index), 2 slim-only (cell = slim index)
//       3 fold (SF3: g = fat index; cell = g mod w, slot = g / w)
template <int D>
struct HashArgs {
  KeySrc keys;
  const uint8_t* ops;
  int64_t n;
  Seeds<D> cell_seeds;
  Seeds<D> slot_seeds;
  Mod cm;  // cell range per row
  Mod zm;  // slot range
  uint32_t row_cells;  // cells per row
  int kb;              // slot bits
  uint32_t fold_w;     // KIND 3: the slim width w
  uint32_t* key_out;
  uint32_t* val_out;
  int unsupported_deletes;  // SF1 / CU: a delete is the failing op
  const uint2* pos;         // SF1 / CU slim pairs: name op t by its key-order position (pos[t].y)
  Ctl* ctl;
};

template <int D, int KIND>
__global__ void __launch_bounds__(256) hash_emit_k(HashArgs<D> a) {
  uint32_t local_fail = NONE32, local_bad = NONE32;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < a.n; t += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = load_key(a.keys, t);
    const uint32_t code = a.ops[t];
    const uint32_t op = code != 0;  // anything but 0 / 1 makes the batch a no-op (t* = 0, below)
    if (code > 1 && local_bad == NONE32) local_bad = (uint32_t)t;
    if (a.unsupported_deletes && op != 0 && local_fail == NONE32) local_fail = (uint32_t)t;
#pragma unroll
    for (int i = 0; i < D; ++i) {
      const uint32_t name = (KIND == 2 && a.pos) ? a.pos[t].y : (uint32_t)t;
      uint32_t cell, v = (name << (a.kb + 1)) | (op << a.kb);
      if (KIND == 3) {
        const uint32_t g = (uint32_t)bucket(key, a.cell_seeds.s[i], a.cm);
        cell = (uint32_t)i * a.fold_w + g % a.fold_w;
        v |= g / a.fold_w;
      } else {
        cell = (uint32_t)i * a.row_cells + (uint32_t)bucket(key, a.cell_seeds.s[i], a.cm);
      }
      if (KIND == 0) v |= (uint32_t)bucket(key, a.slot_seeds.s[i], a.zm);
      a.key_out[(int64_t)i * a.n + t] = cell;
      a.val_out[(int64_t)i * a.n + t] = v;
    }
  }
  // grid-stride order means a thread's first delete is its smallest
  if (local_fail != NONE32) atomicMin(&a.ctl->fail_t, local_fail);
  // a bad op code: report the first one and apply nothing (every op counts as
  // at or after the failing op, so the fat is undone and no run is replayed)
  if (local_bad != NONE32) {
    atomicMin(&a.ctl->bad_op, local_bad);
    atomicMin(&a.ctl->fail_t, 0u);
  }
}

// ---------------------------------------------------------------- 3. segscan
template <int Z>
struct SegState {
  uint32_t flag;  // a segment head lies inside this span
  uint32_t head;  // position of the last head inside the span (if flag)
  int32_t v[Z];   // net count deltas since that head (or over the span)
};

template <int Z>
__device__ __forceinline__ SegState<Z> seg_combine(const SegState<Z>& a, const SegState<Z>& b) {
  if (b.flag) return b;
  SegState<Z> r;
  r.flag = a.flag;
  r.head = a.head;
#pragma unroll
  for (int k = 0; k < Z; ++k) r.v[k] = a.v[k] + b.v[k];
  return r;
}

template <int Z>
__host__ __device__ __forceinline__ SegState<Z> seg_identity() {
  SegState<Z> r;
  r.flag = 0;
  r.head = 0;
#pragma unroll
  for (int k = 0; k < Z; ++k) r.v[k] = 0;
  return r;
}

template <int Z>
struct SegStateOp {
  __device__ __forceinline__ SegState<Z> operator()(const SegState<Z>& a, const SegState<Z>& b) const {
    return seg_combine<Z>(a, b);
  }
};

template <int Z>
__device__ __forceinline__ SegState<Z> shfl_state(const SegState<Z>& s, int src_delta, bool up) {
  SegState<Z> r;
  if (up) {
    r.flag = __shfl_up_sync(0xffffffffu, s.flag, src_delta);
    r.head = __shfl_up_sync(0xffffffffu, s.head, src_delta);
#pragma unroll
    for (int k = 0; k < Z; ++k) r.v[k] = __shfl_up_sync(0xffffffffu, s.v[k], src_delta);
  } else {
    r.flag = __shfl_down_sync(0xffffffffu, s.flag, src_delta);
    r.head = __shfl_down_sync(0xffffffffu, s.head, src_delta);
#pragma unroll
    for (int k = 0; k < Z; ++k) r.v[k] = __shfl_down_sync(0xffffffffu, s.v[k], src_delta);
  }
  return r;
}

// element e as a one-element span
template <int Z, bool HAS_FAT>
__device__ __forceinline__ SegState<Z> elem_state(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals,
                                                  uint32_t e, int kb) {
  SegState<Z> s = seg_identity<Z>();
  const uint32_t c = keys[e];
  s.flag = (e == 0) || (keys[e - 1] != c);
  s.head = e;
  if (HAS_FAT) {
    const uint32_t v = vals[e];
    const uint32_t k = v & ((1u << kb) - 1u);
    const int32_t dl = ((v >> kb) & 1u) ? -1 : 1;
#pragma unroll
    for (int q = 0; q < Z; ++q) s.v[q] = (q == (int)k) ? dl : 0;
  }
  return s;
}

// exclusive block scan of per-thread aggregates (ordered, non-commutative)
template <int Z>
__device__ __forceinline__ SegState<Z> block_exclusive(SegState<Z> agg, SegState<Z>* warp_tot, SegState<Z>* block_tot) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  SegState<Z> inc = agg;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    SegState<Z> o = shfl_state<Z>(inc, off, true);
    if (lane >= off) inc = seg_combine<Z>(o, inc);
  }
  if (lane == 31) warp_tot[wid] = inc;
  __syncthreads();
  if (threadIdx.x == 0) {
    SegState<Z> run = seg_identity<Z>();
    for (int w = 0; w < SCAN_THREADS / 32; ++w) {
      SegState<Z> t = warp_tot[w];
      warp_tot[w] = run;  // exclusive prefix of warp w
      run = seg_combine<Z>(run, t);
    }
    *block_tot = run;
  }
  __syncthreads();
  SegState<Z> excl_in_warp = shfl_state<Z>(inc, 1, true);
  if (lane == 0) excl_in_warp = seg_identity<Z>();
  return seg_combine<Z>(warp_tot[wid], excl_in_warp);
}

template <int Z, bool HAS_FAT>
__global__ void __launch_bounds__(SCAN_THREADS) segscan_reduce_k(const uint32_t* __restrict__ keys,
                                                                 const uint32_t* __restrict__ vals, uint32_t N, int kb,
                                                                 SegState<Z>* __restrict__ tile_agg) {
  __shared__ SegState<Z> warp_tot[SCAN_THREADS / 32];
  __shared__ SegState<Z> block_tot;
  const uint32_t base = blockIdx.x * SCAN_TILE + threadIdx.x * SCAN_ITEMS;
  SegState<Z> agg = seg_identity<Z>();
  if (base + SCAN_ITEMS <= N) {  // vector loads (see sf1_ignore_k)
    uint32_t cc[SCAN_ITEMS], vv[SCAN_ITEMS];
    const uint4* kp = reinterpret_cast<const uint4*>(keys + base);
    const uint4* vp = reinterpret_cast<const uint4*>(vals + base);
#pragma unroll
    for (int h = 0; h < SCAN_ITEMS / 4; ++h) {
      const uint4 a = __ldg(kp + h), b = __ldg(vp + h);
      cc[4 * h] = a.x, cc[4 * h + 1] = a.y, cc[4 * h + 2] = a.z, cc[4 * h + 3] = a.w;
      vv[4 * h] = b.x, vv[4 * h + 1] = b.y, vv[4 * h + 2] = b.z, vv[4 * h + 3] = b.w;
    }
    const uint32_t c_before = base > 0 ? keys[base - 1] : 0u;
#pragma unroll
    for (int q = 0; q < SCAN_ITEMS; ++q) {
      SegState<Z> el = seg_identity<Z>();
      el.flag = (base + q == 0) || (q ? cc[q - 1] : c_before) != cc[q];
      el.head = base + q;
      if (HAS_FAT) {
        const uint32_t k = vv[q] & ((1u << kb) - 1u);
        const int32_t dl = ((vv[q] >> kb) & 1u) ? -1 : 1;
#pragma unroll
        for (int q2 = 0; q2 < Z; ++q2) el.v[q2] = (q2 == (int)k) ? dl : 0;
      }
      agg = seg_combine<Z>(agg, el);
    }
  } else {
#pragma unroll
    for (int q = 0; q < SCAN_ITEMS; ++q) {
      uint32_t e = base + q;
      if (e < N) agg = seg_combine<Z>(agg, elem_state<Z, HAS_FAT>(keys, vals, e, kb));
    }
  }
  (void)block_exclusive<Z>(agg, warp_tot, &block_tot);
  if (threadIdx.x == 0) tile_agg[blockIdx.x] = block_tot;
}



struct ScanOut {
  const uint32_t* fat_init;  // snapshot of the fat (cell-major, Z per cell)
  uint32_t* fat_out;         // final fat (written at segment ends)
  uint32_t* obs;             // WRITE_OBS 1: [t*D + row] post own count / bucket max; 4: [t] min over rows (b_min)
  uint2* obs2;               // [t*D + row]: {own slot count after the op, max of the other slots}
  uint2* links;              // [t*D + row]: {rank of the op in its cell, previous op on the cell or NONE}
  uint32_t n;                // ops
  uint32_t D;
  uint32_t row_cells;
  Ctl* ctl;
  uint32_t* tkey;            // WRITE_OBS 6: [e] the op t of sorted element e
  uint32_t* tval;            //   and its post-op own fat count (b_min candidates, min-reduced per op later)
};

// WRITE_OBS: 0 none, 1 obs (b_min / bucket max), 2 obs2 (own count, max of the others),
//            3 obs2 (own count, sum of the others clamped to 2^32 - 1: the SF2/SF3/SF4 trigger)
//            5 obs (CU drop pass: 1 + an upper bound of each op's minimum; fat_init = the slim)
//            6 tkey / tval (SF1 / SF2 b_min: (t, post-op own count) per element in cell order,
//              coalesced; bmin_from_pairs reduces them per op)
template <int Z, bool HAS_FAT, int WRITE_OBS, bool WRITE_LINKS>
__global__ void __launch_bounds__(SCAN_THREADS) segscan_apply_k(const uint32_t* __restrict__ keys,
                                                                const uint32_t* __restrict__ vals, uint32_t N, int kb,
                                                                const SegState<Z>* __restrict__ carry, ScanOut o) {
  __shared__ SegState<Z> warp_tot[SCAN_THREADS / 32];
  __shared__ SegState<Z> block_tot;
  const uint32_t base = blockIdx.x * SCAN_TILE + threadIdx.x * SCAN_ITEMS;
  // this thread's elements, staged in registers once: cell, value, segment
  // head / end flags, and (fat kinds) the cell's fat snapshot; the snapshot
  // loads are issued before the block scan so their latency overlaps it
  uint32_t cc[SCAN_ITEMS], vv[SCAN_ITEMS];
  if (base + SCAN_ITEMS <= N) {
    const uint4* kp = reinterpret_cast<const uint4*>(keys + base);
    const uint4* vp = reinterpret_cast<const uint4*>(vals + base);
#pragma unroll
    for (int h = 0; h < SCAN_ITEMS / 4; ++h) {
      const uint4 a = __ldg(kp + h), b = __ldg(vp + h);
      cc[4 * h] = a.x, cc[4 * h + 1] = a.y, cc[4 * h + 2] = a.z, cc[4 * h + 3] = a.w;
      vv[4 * h] = b.x, vv[4 * h + 1] = b.y, vv[4 * h + 2] = b.z, vv[4 * h + 3] = b.w;
    }
  } else {
#pragma unroll
    for (int q = 0; q < SCAN_ITEMS; ++q) {
      cc[q] = base + q < N ? keys[base + q] : U32MAX;
      vv[q] = base + q < N ? vals[base + q] : 0u;
    }
  }
  const bool has_prev = base > 0 && base < N;
  const uint32_t c_before = has_prev ? keys[base - 1] : 0u;
  const uint32_t t_before = has_prev ? (vals[base - 1] >> (kb + 1)) : NONE32;
  const bool has_next = base + SCAN_ITEMS < N;
  const uint32_t c_after = has_next ? keys[base + SCAN_ITEMS] : 0u;
  uint32_t init[HAS_FAT ? SCAN_ITEMS : 1][HAS_FAT ? Z : 1];
  if (HAS_FAT) {
#pragma unroll
    for (int q = 0; q < SCAN_ITEMS; ++q) {
      if (base + q < N) {
        if (Z == 4) {
          const uint4 f = __ldg(reinterpret_cast<const uint4*>(o.fat_init) + cc[q]);
          init[q][0] = f.x, init[q][1 % Z] = f.y, init[q][2 % Z] = f.z, init[q][3 % Z] = f.w;
        } else {
#pragma unroll
          for (int q2 = 0; q2 < Z; ++q2) init[q][q2] = __ldg(o.fat_init + (size_t)cc[q] * Z + q2);
        }
      } else {
#pragma unroll
        for (int q2 = 0; q2 < Z; ++q2) init[q][q2] = 0u;
      }
    }
  }
  bool hd[SCAN_ITEMS];
#pragma unroll
  for (int q = 0; q < SCAN_ITEMS; ++q) hd[q] = (base + q == 0) || (q ? cc[q - 1] : c_before) != cc[q];
  auto elem = [&](int q) {
    SegState<Z> s = seg_identity<Z>();
    s.flag = hd[q] ? 1u : 0u;
    s.head = base + q;
    if (HAS_FAT) {
      const uint32_t k = vv[q] & ((1u << kb) - 1u);
      const int32_t dl = ((vv[q] >> kb) & 1u) ? -1 : 1;
#pragma unroll
      for (int q2 = 0; q2 < Z; ++q2) s.v[q2] = (q2 == (int)k) ? dl : 0;
    }
    return s;
  };
  SegState<Z> agg = seg_identity<Z>();
#pragma unroll
  for (int q = 0; q < SCAN_ITEMS; ++q)
    if (base + q < N) agg = seg_combine<Z>(agg, elem(q));
  SegState<Z> run = block_exclusive<Z>(agg, warp_tot, &block_tot);
  run = seg_combine<Z>(carry[blockIdx.x], run);
  uint32_t local_fail = NONE32;
  uint32_t prev_t = t_before;
#pragma unroll
  for (int q = 0; q < SCAN_ITEMS; ++q) {
    const uint32_t e = base + q;
    if (e >= N) break;
    run = seg_combine<Z>(run, elem(q));
    const uint32_t c = cc[q];
    const uint32_t v = vv[q];
    const uint32_t t = v >> (kb + 1);
    const uint32_t op = (v >> kb) & 1u;
    const uint32_t row = c / o.row_cells;
    uint32_t rec_own = 0, rec_oth = 0;  // observations carried in the link record
    if (HAS_FAT) {
      const uint32_t k = v & ((1u << kb) - 1u);
      uint32_t own_init = init[q][0];
#pragma unroll
      for (int q2 = 1; q2 < Z; ++q2)
        if (q2 == (int)k) own_init = init[q][q2];
      int32_t own_d = run.v[0];
#pragma unroll
      for (int q2 = 1; q2 < Z; ++q2)
        if (q2 == (int)k) own_d = run.v[q2];
      const int64_t post_own = (int64_t)own_init + (int64_t)own_d;
      const int64_t pre_own = post_own + (op ? 1 : -1);
      if (op == 0 ? (pre_own == (int64_t)U32MAX) : (pre_own == 0)) local_fail = min(local_fail, t);
      if (WRITE_OBS == 2 || WRITE_OBS == 3) {
        uint32_t others = 0;
        if (WRITE_OBS == 2) {
#pragma unroll
          for (int q2 = 0; q2 < Z; ++q2)
            if (q2 != (int)k) others = max(others, (uint32_t)((int64_t)init[q][q2] + run.v[q2]));
        } else {
          uint64_t sum = 0;
#pragma unroll
          for (int q2 = 0; q2 < Z; ++q2)
            if (q2 != (int)k) sum += (uint64_t)((int64_t)init[q][q2] + run.v[q2]);
          others = (uint32_t)min(sum, (uint64_t)U32MAX);
        }
        if (WRITE_LINKS) {
          rec_own = (uint32_t)post_own;
          rec_oth = others;
        } else {
          o.obs2[(size_t)t * o.D + row] = make_uint2((uint32_t)post_own, others);
        }
      }
      if (WRITE_OBS == 6) {
        o.tkey[e] = t;
        o.tval[e] = (uint32_t)min(post_own, (int64_t)U32MAX);
      }
      if (WRITE_OBS == 4) {
        // b_min of op t = min over its d rows of the post-op own fat count:
        // one 4-B atomicMin per (op, row) into a per-op word (a scattered
        // 4-B store per (op, row) would cost L2 a DRAM fill per sector)
        atomicMin(o.obs + t, (uint32_t)min(post_own, (int64_t)U32MAX));
      }
      if (WRITE_OBS == 1) {
        uint32_t ob;
        if (op == 0) {
          ob = (uint32_t)post_own;
        } else {
          ob = 0;
#pragma unroll
          for (int q2 = 0; q2 < Z; ++q2) ob = max(ob, (uint32_t)((int64_t)init[q][q2] + run.v[q2]));
        }
        o.obs[(size_t)t * o.D + row] = ob;
      }
      const bool last = (e + 1 == N) || ((q + 1 < SCAN_ITEMS) ? cc[q + 1 < SCAN_ITEMS ? q + 1 : q] : c_after) != c;
      if (last) {
#pragma unroll
        for (int q2 = 0; q2 < Z; ++q2) o.fat_out[(size_t)c * Z + q2] = (uint32_t)((int64_t)init[q][q2] + run.v[q2]);
      }
    }
    if (WRITE_OBS == 5) {
      // CU: 1 + (the cell's value before the batch + the ops before this one
      // on it), min over the op's rows = 1 + an upper bound of its minimum
      const unsigned long long ub = (unsigned long long)__ldg(o.fat_init + c) + (e - run.head) + 1ull;
      atomicMin(o.obs + t, (uint32_t)min(ub, (unsigned long long)U32MAX));
    }
    if (WRITE_LINKS) {
      // One 32-B record per (op, row): rank in the cell, previous op,
      // observations, the cell and the op's sorted position (row 0: its
      // row-0 order index). Whole-sector scattered stores: a 16-B store into
      // a sector written at another time costs L2 a DRAM fill.
      const uint32_t prev = (e > run.head) ? prev_t : NONE32;
      uint4* rec = reinterpret_cast<uint4*>(o.links) + ((size_t)t * o.D + row) * 2;
      st_sector(rec, make_uint4(e - run.head, prev, rec_own, rec_oth), make_uint4(c, e, 0u, 0u));
    }
    prev_t = t;
  }
  (void)has_next;
  if (HAS_FAT && local_fail != NONE32) atomicMin(&o.ctl->fail_t, local_fail);
}


// ---------------------------------------------------------------- SF1 / SF2: b_min per op
// b_min of op t = min over its d rows of its post-op own fat count. The fat
// scan runs in cell order, so the d candidates of an op sit at random
// places; rather than a 4-B atomicMin per (op, row) into a per-op array far
// larger than L2 (every atomic a DRAM sector fill and write-back: cfg 4's
// scan moved 34.7 GB), the scan writes (t, candidate) pairs in place, a
// partial radix sort on t's bits above BMIN_BITS groups them into ranges of
// 2^BMIN_BITS consecutive ops (every op has exactly d pairs, so range b
// starts at pair d b 2^BMIN_BITS), and one CTA per range takes the minima in
// shared memory.
constexpr int BMIN_BITS = 13;
__global__ void __launch_bounds__(512) bmin_bucket_k(const uint32_t* __restrict__ tkey, const uint32_t* __restrict__ tval,
                                                     uint32_t n, uint32_t d, uint32_t* __restrict__ obs) {
  __shared__ uint32_t bm[1 << BMIN_BITS];
  const uint32_t t0 = blockIdx.x << BMIN_BITS, cnt = min(n - t0, 1u << BMIN_BITS);
  for (uint32_t i = threadIdx.x; i < cnt; i += blockDim.x) bm[i] = U32MAX;
  __syncthreads();
  const size_t p1 = ((size_t)t0 + cnt) * d;
  for (size_t p = (size_t)t0 * d + threadIdx.x; p < p1; p += blockDim.x) atomicMin(bm + (tkey[p] - t0), tval[p]);
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < cnt; i += blockDim.x) obs[t0 + i] = bm[i];
}

// ---------------------------------------------------------------- SF1 / CU: ignorable (op, row) pairs
// An SF1 slim cell never drops below the batch net count of any key that maps
// to it: inserts only raise cells, and a key's own inserts keep the min of its
// d cells at or above its count (b_min >= its count, and each insert raises a
// min below b_min by one). So when an earlier op of the batch on the same cell
// belongs to a key whose count then was >= this op's b_min, the cell is >=
// b_min at this op's turn: it is neither a min below b_min nor raised, and the
// op's outcome does not depend on it. Such (op, row) pairs leave the cell's
// sequence: the engine neither waits for nor publishes them. Any row may be
// dropped; runs are then laid out in key order (runs_head_k, key_prev_k).
// CU reuses the pass with "b_min" = 1 + an upper bound of the op's minimum
// (segscan WRITE_OBS 5): a row whose lower bound exceeds it is not a minimum.

// per-op count of its key among the batch's ops up to and including it
__global__ void iota_k(uint32_t* __restrict__ t, uint32_t n) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) t[j] = j;
}
template <typename K>
__global__ void key_heads_k(const K* __restrict__ ks, uint32_t n, uint32_t* __restrict__ headpos) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
    headpos[j] = (j == 0 || ks[j] != ks[j - 1]) ? j : 0u;
}
// 64-bit keys: a group id per op from an open-addressing table (linear
// probing, one CAS per distinct key), so the stable key grouping sorts
// ceil(log2(cap + 1) / 8) passes of 4-B ids instead of 8 passes of 8-B keys.
// Ids are table slots (the key ~0, the empty mark, gets the id cap); group
// order varies between runs, grouping does not, and nothing downstream
// depends on the order of the groups.
constexpr unsigned long long SLOT_EMPTY = ~0ull;
__global__ void key_slot_k(const uint64_t* __restrict__ keys, uint32_t n, unsigned long long* __restrict__ table,
                           uint32_t cap, uint32_t* __restrict__ slot) {
  const uint32_t mask = cap - 1u;
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const unsigned long long k = keys[t];
    uint32_t s = cap;
    if (k != SLOT_EMPTY) {
      s = (uint32_t)(mix64(k ^ 0x2545F4914F6CDD1Dull) >> 32) & mask;
      while (true) {
        const unsigned long long cur = *reinterpret_cast<volatile const unsigned long long*>(table + s);
        if (cur == k) break;
        if (cur == SLOT_EMPTY) {
          const unsigned long long prev = atomicCAS(table + s, SLOT_EMPTY, k);
          if (prev == SLOT_EMPTY || prev == k) break;
        }
        s = (s + 1u) & mask;
      }
    }
    slot[t] = s;
  }
}
static uint32_t slot_cap(uint32_t n) {  // a power of two >= 1.25 n (load <= 0.8 with every key distinct)
  uint64_t c = 1024;
  while (c < (uint64_t)n + n / 4) c <<= 1;
  return (uint32_t)c;
}

// per op in key order, 16 B gathered once by the ignore scan: {key count,
// b_min, the key's previous op (j - 1, or NONE32), the op t}; b_min is laid
// out by t (SF1: the fat phase) or already by j (CU: the upper-bound scan)
__global__ void cb_pack_k(const uint32_t* __restrict__ tb, const uint32_t* __restrict__ headpos,
                          const uint32_t* __restrict__ bmin, int bmin_by_j, uint32_t n, uint4* __restrict__ cb) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const uint32_t t = tb[j], h = headpos[j];
    cb[j] = make_uint4(j - h + 1u, bmin[bmin_by_j ? j : t], h == j ? NONE32 : j - 1u, t);
  }
}

// key order -> op order: {count of the op's key up to and including it, the
// op's position j in the key-sorted list} in one 8-B store per op. The
// dropped-pair pipeline names ops by j: a key's ops are consecutive there,
// so its previous op is j - 1 and per-op data laid out by j is read with
// locality wherever a cell's sequence follows one key.
// (four positions per thread and iteration, loads first: the scattered
// stores are partial sectors, and one position at a time left the kernel
// latency-bound at 2 % issue)
template <typename K>
__global__ void key_meta_k(const K* __restrict__ ks, const uint32_t* __restrict__ tb,
                           const uint32_t* __restrict__ headpos, uint32_t n, uint2* __restrict__ meta) {
  constexpr int U = 4;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t j0 = blockIdx.x * blockDim.x + threadIdx.x; j0 < n; j0 += U * stride) {
    uint32_t t[U], c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t j = j0 + u * stride;
      if (j < n) {
        t[u] = tb[j];
        c[u] = j - headpos[j] + 1u;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (j0 + u * stride < n) meta[t[u]] = make_uint2(c[u], j0 + u * stride);
  }
}

struct SegMax {
  uint32_t flag, v;
};
struct SegMaxOp {
  __device__ __forceinline__ SegMax operator()(const SegMax& a, const SegMax& b) const {
    return SegMax{a.flag | b.flag, b.flag ? b.v : max(a.v, b.v)};
  }
};

// ignore flags in sorted (cell) order: within a 2048-element tile, the
// segmented prefix max of the key counts of earlier ops on the cell (a valid
// lower bound of the cell; earlier tiles are simply not consulted)
__global__ void __launch_bounds__(SCAN_THREADS) sf1_ignore_k(const uint32_t* __restrict__ keys,
                                                            const uint32_t* __restrict__ vals, uint32_t N,
                                                            uint32_t row_cells, const uint4* __restrict__ cb,
                                                            const Ctl* __restrict__ ctl, uint8_t* __restrict__ ign,
                                                            uint32_t* __restrict__ kpc, uint32_t* __restrict__ dmask) {
  typedef cub::BlockScan<SegMax, SCAN_THREADS> BS;
  __shared__ typename BS::TempStorage tmp;
  const uint32_t tstar = ctl->fail_t;
  const uint32_t base = blockIdx.x * SCAN_TILE + threadIdx.x * SCAN_ITEMS;
  // this thread's elements, loaded once: cell, head flag, the op's key-order
  // position j, and {count, b_min, previous op (j space), t} gathered by j
  // (vector loads: a warp reads 1 KB of cells and values contiguously; the
  // scalar strided loads they replace re-requested every sector 8 times,
  // and the gathers below evicted them from L1 and L2 in between)
  uint32_t cc[SCAN_ITEMS], tt[SCAN_ITEMS];
  uint4 kb[SCAN_ITEMS];
  bool hd[SCAN_ITEMS];
  if (base + SCAN_ITEMS <= N) {
    const uint4* kp = reinterpret_cast<const uint4*>(keys + base);
    const uint4* vp = reinterpret_cast<const uint4*>(vals + base);
#pragma unroll
    for (int h = 0; h < SCAN_ITEMS / 4; ++h) {
      const uint4 a = __ldg(kp + h), b = __ldg(vp + h);
      cc[4 * h] = a.x, cc[4 * h + 1] = a.y, cc[4 * h + 2] = a.z, cc[4 * h + 3] = a.w;
      tt[4 * h] = b.x >> 1, tt[4 * h + 1] = b.y >> 1, tt[4 * h + 2] = b.z >> 1, tt[4 * h + 3] = b.w >> 1;
    }
  } else {
#pragma unroll
    for (int q = 0; q < SCAN_ITEMS; ++q) {
      cc[q] = base + q < N ? keys[base + q] : U32MAX;
      tt[q] = base + q < N ? vals[base + q] >> 1 : 0u;
    }
  }
  const uint32_t c_before = (base > 0 && base < N) ? keys[base - 1] : 0u;
#pragma unroll
  for (int q = 0; q < SCAN_ITEMS; ++q)
    hd[q] = base + q < N && (base + q == 0 || (q ? cc[q - 1] : c_before) != cc[q]);
#pragma unroll
  for (int q = 0; q < SCAN_ITEMS; ++q) kb[q] = base + q < N ? __ldg(cb + tt[q]) : make_uint4(0u, 0u, 0u, 0u);
  SegMax agg{0u, 0u};
  SegMaxOp op;
#pragma unroll
  for (int q = 0; q < SCAN_ITEMS; ++q) {
    if (base + q < N) {
      const SegMax el{hd[q] ? 1u : 0u, kb[q].x};
      agg = q == 0 ? el : op(agg, el);
    }
  }
  SegMax run;
  BS(tmp).ExclusiveScan(agg, run, SegMax{0u, 0u}, op);
  if (threadIdx.x == 0) run = SegMax{0u, 0u};
  uint32_t flags[2] = {0u, 0u};
#pragma unroll
  for (int q = 0; q < SCAN_ITEMS; ++q) {
    const uint32_t lb = hd[q] ? 0u : run.v;
    if (base + q < N && kb[q].w < tstar && lb >= kb[q].y) {
      flags[q >> 2] |= 1u << (8 * (q & 3));
      // the op's dropped rows, one byte per op (D <= 8), by key-order position
      const uint32_t j = tt[q], row = cc[q] / row_cells;
      atomicOr(dmask + (j >> 2), 1u << (8 * (j & 3) + row));
    }
    run = op(run, SegMax{hd[q] ? 1u : 0u, kb[q].x});
  }
  static_assert(SCAN_ITEMS == 8, "one 8-B store of the flags");
  if (base + SCAN_ITEMS <= N) {
    *reinterpret_cast<uint2*>(ign + base) = make_uint2(flags[0], flags[1]);
    uint4* kp = reinterpret_cast<uint4*>(kpc + base);
    kp[0] = make_uint4(kb[0].z, kb[1].z, kb[2].z, kb[3].z);
    kp[1] = make_uint4(kb[4].z, kb[5].z, kb[6].z, kb[7].z);
  } else {
#pragma unroll
    for (int q = 0; q < SCAN_ITEMS; ++q)
      if (base + q < N) {
        ign[base + q] = (uint8_t)((flags[q >> 2] >> (8 * (q & 3))) & 1u);
        kpc[base + q] = kb[q].z;
      }
  }
}

// filtered links: for every element, the number of non-ignored elements
// before it in its cell (its rank in the cell's filtered sequence) and the
// last non-ignored op before it; a segmented scan (reduce / tile carry /
// apply) like segscan, over {segment-head flag, count, last op}
struct SegCnt {
  uint32_t flag, cnt, last;
};
struct SegCntOp {
  __device__ __forceinline__ SegCnt operator()(const SegCnt& a, const SegCnt& b) const {
    if (b.flag) return b;
    return SegCnt{a.flag, a.cnt + b.cnt, b.last != NONE32 ? b.last : a.last};
  }
};
// a thread's SCAN_ITEMS consecutive elements, staged in registers once:
// cell, op, dropped flag, and the elements' {head, kept, op} scan states
struct FiltItems {
  uint32_t c[SCAN_ITEMS], t[SCAN_ITEMS];
  uint32_t ign;  // bit q: element q is dropped
  uint32_t hd;   // bit q: element q heads its cell's segment
};
__device__ __forceinline__ void filt_load(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals,
                                          const uint8_t* __restrict__ ign, uint32_t N, uint32_t base, FiltItems& it) {
  uint32_t vv[SCAN_ITEMS];
  it.ign = 0;
  if (base + SCAN_ITEMS <= N) {
    const uint4* kp = reinterpret_cast<const uint4*>(keys + base);
    const uint4* vp = reinterpret_cast<const uint4*>(vals + base);
#pragma unroll
    for (int h = 0; h < SCAN_ITEMS / 4; ++h) {
      const uint4 a = __ldg(kp + h), b = __ldg(vp + h);
      it.c[4 * h] = a.x, it.c[4 * h + 1] = a.y, it.c[4 * h + 2] = a.z, it.c[4 * h + 3] = a.w;
      vv[4 * h] = b.x, vv[4 * h + 1] = b.y, vv[4 * h + 2] = b.z, vv[4 * h + 3] = b.w;
    }
    static_assert(SCAN_ITEMS == 8, "one 8-B load of the dropped flags");
    const uint2 g = __ldg(reinterpret_cast<const uint2*>(ign + base));
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      it.ign |= ((g.x >> (8 * q)) & 1u) << q;
      it.ign |= ((g.y >> (8 * q)) & 1u) << (q + 4);
    }
  } else {
#pragma unroll
    for (int q = 0; q < SCAN_ITEMS; ++q) {
      const bool in = base + q < N;
      it.c[q] = in ? keys[base + q] : U32MAX;
      vv[q] = in ? vals[base + q] : 0u;
      if (in && ign[base + q]) it.ign |= 1u << q;
    }
  }
  const uint32_t c_before = (base > 0 && base < N) ? keys[base - 1] : 0u;
  it.hd = 0;
#pragma unroll
  for (int q = 0; q < SCAN_ITEMS; ++q) {
    it.t[q] = vv[q] >> 1;
    if (base + q == 0 || (q ? it.c[q - 1] : c_before) != it.c[q]) it.hd |= 1u << q;
  }
}
__device__ __forceinline__ SegCnt filt_elem(const FiltItems& it, int q) {
  const bool keep = !((it.ign >> q) & 1u);
  return SegCnt{(it.hd >> q) & 1u, keep ? 1u : 0u, keep ? it.t[q] : NONE32};
}
__global__ void __launch_bounds__(SCAN_THREADS) filt_reduce_k(const uint32_t* __restrict__ keys,
                                                             const uint32_t* __restrict__ vals,
                                                             const uint8_t* __restrict__ ign, uint32_t N,
                                                             SegCnt* __restrict__ tile_agg) {
  typedef cub::BlockScan<SegCnt, SCAN_THREADS> BS;
  __shared__ typename BS::TempStorage tmp;
  const uint32_t base = blockIdx.x * SCAN_TILE + threadIdx.x * SCAN_ITEMS;
  FiltItems it;
  filt_load(keys, vals, ign, N, base, it);
  SegCntOp op;
  SegCnt agg{0u, 0u, NONE32};
#pragma unroll
  for (int q = 0; q < SCAN_ITEMS; ++q)
    if (base + q < N) agg = op(agg, filt_elem(it, q));
  // ordered (non-commutative): the block's inclusive scan, last thread's value
  SegCnt inc, tot;
  BS(tmp).InclusiveScan(agg, inc, op, tot);
  if (threadIdx.x == 0) tile_agg[blockIdx.x] = tot;
}
// Two passes over the filtered sequence (same scan state as filt_reduce_k):
// filt_brk_k marks op t as a run break when one of its kept pairs follows a
// kept op other than the key's previous op (kpc, from the ignore scan), one
// bit per op; runs_head_ign_k decides the run heads from those bits and the
// dropped-row bytes; filt_rec_k then writes the 32-B link record of the kept
// pairs of run heads only (the rest of the pipeline reads no other). Every
// (op, row) record used to be written: 400M scattered sectors at cfg 4.
template <bool REC>
__global__ void __launch_bounds__(SCAN_THREADS) filt_apply_k(const uint32_t* __restrict__ keys,
                                                            const uint32_t* __restrict__ vals,
                                                            const uint8_t* __restrict__ ign, uint32_t N, uint32_t D,
                                                            uint32_t row_cells, const SegCnt* __restrict__ carry,
                                                            const uint32_t* __restrict__ kpc,
                                                            const uint32_t* __restrict__ tb,
                                                            uint32_t* __restrict__ bits, uint4* __restrict__ links) {
  typedef cub::BlockScan<SegCnt, SCAN_THREADS> BS;
  __shared__ typename BS::TempStorage tmp;
  SegCntOp op;
  const uint32_t base = blockIdx.x * SCAN_TILE + threadIdx.x * SCAN_ITEMS;
  FiltItems it;
  filt_load(keys, vals, ign, N, base, it);
  uint32_t kp[SCAN_ITEMS];
  if (!REC) {
    if (base + SCAN_ITEMS <= N) {
      const uint4 a = __ldg(reinterpret_cast<const uint4*>(kpc + base));
      const uint4 b = __ldg(reinterpret_cast<const uint4*>(kpc + base) + 1);
      kp[0] = a.x, kp[1] = a.y, kp[2] = a.z, kp[3] = a.w, kp[4] = b.x, kp[5] = b.y, kp[6] = b.z, kp[7] = b.w;
    } else {
#pragma unroll
      for (int q = 0; q < SCAN_ITEMS; ++q) kp[q] = base + q < N ? kpc[base + q] : NONE32;
    }
  }
  SegCnt agg{0u, 0u, NONE32};
#pragma unroll
  for (int q = 0; q < SCAN_ITEMS; ++q)
    if (base + q < N) agg = op(agg, filt_elem(it, q));
  SegCnt run;
  BS(tmp).ExclusiveScan(agg, run, SegCnt{0u, 0u, NONE32}, op);
  if (threadIdx.x == 0) run = SegCnt{0u, 0u, NONE32};
  run = op(carry[blockIdx.x], run);
#pragma unroll
  for (int q = 0; q < SCAN_ITEMS; ++q) {
    const uint32_t e = base + q;
    if (e >= N) break;
    const uint32_t c = it.c[q], j = it.t[q];  // ops named by key-order position j (see key_meta_k)
    const SegCnt el = filt_elem(it, q);
    const SegCnt before = el.flag ? SegCnt{1u, 0u, NONE32} : run;
    const bool kept = !((it.ign >> q) & 1u);
    if (!REC) {
      if (kept && before.last != kp[q]) atomicOr(bits + (j >> 5), 1u << (j & 31));
    } else if (kept && ((__ldg(bits + (j >> 5)) >> (j & 31)) & 1u)) {  // run heads, by j
      const uint32_t t = __ldg(tb + j);
      uint4* rec = links + ((size_t)t * D + c / row_cells) * 2;
      st_sector(rec, make_uint4(before.cnt, before.last, 0u, 0u), make_uint4(c, e, 0u, 0u));
    }
    run = op(run, el);
  }
}

// run heads of the key-ordered SF1 / CU runs (the semantics of runs_head_k
// with dropped pairs): op t (key-order position j) continues the key's
// previous op j - 1 when it is valid, keeps a row, drops the same rows as
// j - 1, and no kept pair of t follows anything but j - 1 in its cell (no
// break bit at j). Heads are written by t: run ids follow stream order.
__global__ void runs_head_ign_k(uint32_t n, const Ctl* __restrict__ ctl, const uint8_t* __restrict__ dmask,
                                const uint32_t* __restrict__ brk, const uint2* __restrict__ kmeta, uint32_t D,
                                uint32_t* __restrict__ headflag, uint32_t* __restrict__ headbits,
                                uint32_t* __restrict__ headbits_j) {
  const uint32_t tstar = ctl->fail_t, full = (1u << D) - 1u;
  const uint32_t stride = gridDim.x * blockDim.x;
  const uint32_t n32 = (n + 31) & ~31u;  // whole warps, so every ballot covers one word of bits
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < n32; t += stride) {
    bool head = false;
    if (t < n) {
      const bool valid = t < tstar;
      const uint2 km = kmeta[t];  // {key count, j}: a count above 1 means j - 1 is the key's previous op
      const uint32_t j = km.y;
      const uint32_t m = dmask[j];
      bool cont = valid && m != full && km.x > 1u && !((__ldg(brk + (j >> 5)) >> (j & 31)) & 1u);
      if (cont) cont = dmask[j - 1] == m;
      head = valid && !cont;
      headflag[t] = head ? 1u : 0u;
      if (head) atomicOr(headbits_j + (j >> 5), 1u << (j & 31));  // (heads are few)
    }
    const unsigned hb = __ballot_sync(0xffffffffu, head);
    if ((threadIdx.x & 31) == 0) headbits[t >> 5] = hb;
  }
}

// ---------------------------------------------------------------- 4. runs
template <int D>
struct RunArgs {
  const uint32_t* vals0;  // row-0 sorted vals (slim cells)
  int kb;
  uint32_t n;
  const uint2* links;      // {rank in cell, prev op} per (t, row), every lstride-th uint2
  int lstride;
  const uint32_t* obs;     // SF1/SF2: b_min per op [t] (segscan WRITE_OBS 4); null otherwise
  KeySrc keys;
  uint8_t* opflags;        // [e]: bit0 delete, bit1 continues the run, bit2 valid (t < t*)
  uint32_t* opdata;        // SF1: b_min per op, row-0 order
  uint32_t* headflag;      // [t] (written by runs_head_k)
  const uint32_t* order;   // key order (ignore pass): run extents are positions in the key-sorted op list
  int obs_by_pos;          // obs is laid out by key-order position (CU's upper bounds), not by op
  const uint4* cbk;        // key order: the ignore pass's {count, b_min, prev, t} per position (b_min read coalesced)
  const uint32_t* hbits;   // key order: run heads as bits per op (an L2-resident copy of headflag)
  uint32_t* delbits;       // [e / 32] bit e % 32: op e (row-0 order) is a delete; may be null
  uint32_t* bnd;           // [e]: 1 if op e does not continue the run before it (run start or invalid)
  uint32_t* isdel;         // [e]: 1 if op e is a delete (scanned into delete prefix counts)
  Ctl* ctl;
};

// Run heads in stream order (coalesced over t): op t continues the run
// before it when all its d cells were last touched by the same op, of the
// same key (the closed forms need the same key, not just the same cells).
template <int D>
__global__ void __launch_bounds__(256) runs_head_k(RunArgs<D> a) {
  const uint32_t tstar = a.ctl->fail_t;
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < a.n; t += gridDim.x * blockDim.x) {
    const bool valid = t < tstar;
    // every row's previous op is the same op p, of the same key
    uint32_t p = NONE32;
    bool cont = valid;
#pragma unroll
    for (int i = 0; i < D; ++i) {
      const uint32_t prev = a.links[((size_t)t * D + i) * 4].y;
      if (prev == NONE32) cont = false;
      else if (p == NONE32) p = prev;
      else if (prev != p) cont = false;
    }
    cont = cont && p != NONE32 && load_key(a.keys, p) == load_key(a.keys, t);
    a.headflag[t] = (valid && !cont) ? 1u : 0u;
  }
}


// Per op in row-0 order: flags, b_min (SF1/SF2), delete bits, run boundaries.
template <int D>
__global__ void __launch_bounds__(256) runs_mark_k(RunArgs<D> a) {
  const uint32_t tstar = a.ctl->fail_t;
  uint32_t ins = 0;
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < a.n; e += gridDim.x * blockDim.x) {
    // position e: row-0 order, or key order (SF1 / CU with dropped rows: every
    // valid op is an insert there, a delete being the failing op)
    const uint32_t v = a.order ? 0u : a.vals0[e];
    const uint32_t t = a.order ? a.order[e] : v >> (a.kb + 1);
    const bool valid = t < tstar;
    const uint32_t op = a.order ? (valid ? 0u : 1u) : (v >> a.kb) & 1u;
    const bool cont = valid && !(a.hbits ? ((__ldg(a.hbits + (t >> 5)) >> (t & 31)) & 1u) : a.headflag[t]);
    a.opflags[e] = (uint8_t)(op | (cont ? 2u : 0u) | (valid ? 4u : 0u));
    if (a.obs) a.opdata[e] = a.cbk ? a.cbk[e].y : a.obs[a.obs_by_pos ? e : t];  // per-op b_min / cap
    if (a.delbits) {
      // e advances in warp-aligned strides, so the ballot covers one word
      const unsigned bits = __ballot_sync(__activemask(), op != 0);
      if ((threadIdx.x & 31) == 0) a.delbits[e >> 5] = bits;
    }
    a.bnd[e] = cont ? 0u : 1u;
    a.isdel[e] = op;
    if (valid && op == 0) ++ins;
  }
  // n_ins: warp reduce then one atomic per warp
  for (int off = 16; off > 0; off >>= 1) ins += __shfl_down_sync(0xffffffffu, ins, off);
  if ((threadIdx.x & 31) == 0 && ins) atomicAdd(&a.ctl->n_ins, (unsigned long long)ins);
}

// Run records, indexed by run id (= rank of the head in stream order): where
// the run starts in row-0 order, its length (+ a has-delete bit), its d slim
// cells, the head's rank in each cell (the cell's sequence number the run
// must wait for) and, for SFF, the key's own slot count before the run (A)
// and the maximum of the other slots of the bucket (O) in every row.
template <int D>
struct SFK_RUNREC_ALIGN RunRec {  // whole 32-B sectors (full-sector stores, vector loads)
  uint32_t e0, info;
  uint32_t bits0;  // SFF: delete flags of the run's first 32 ops
  uint32_t cells[D];
  uint32_t rank[D];
  uint32_t A[D];
  uint32_t O[D];
};

template <int D>
struct BuildArgs {
  const uint32_t* headflag;
  const uint32_t* ridx;
  const uint8_t* opflags;
  const uint32_t* bidx;     // exclusive prefix count of boundaries (row-0 order)
  const uint32_t* bpos;     // position of the k-th boundary; bpos[K] = n
  const uint32_t* delpre;   // exclusive prefix count of deletes, n + 1 entries
  const uint32_t* delbits;  // SFF
  const uint2* obs2;        // SFF
  const uint2* links;
  int lstride;              // 4 when links, obs2 and the cell share one 32-B record per (t, row)
  uint32_t n;
  KeySrc keys;
  Seeds<D> seeds;
  Mod wm;
  uint32_t w;
  RunRec<D>* recs;
  const uint32_t* order;    // key order (see RunArgs)
  const uint8_t* dmask;     // key order: the dropped rows of each op (link records exist for kept rows of heads only)
  const uint32_t* hbits;    // key order: run heads as bits per op
  Ctl* ctl;
};

__global__ void boundary_pos_k(const uint32_t* __restrict__ bnd, const uint32_t* __restrict__ bidx, uint32_t n,
                               uint32_t* __restrict__ bpos) {
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    if (bnd[e]) bpos[bidx[e]] = e;
    if (e == n - 1) bpos[bidx[e] + bnd[e]] = n;
  }
}

template <int D>
__global__ void __launch_bounds__(256) runs_build_k(BuildArgs<D> a) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < a.n; j += gridDim.x * blockDim.x) {
    if (j == a.n - 1) a.ctl->n_runs = a.ridx[j] + a.headflag[j];
    const uint32_t t = a.order ? a.order[j] : j;
    if (!(a.hbits ? ((__ldg(a.hbits + (t >> 5)) >> (t & 31)) & 1u) : a.headflag[t])) continue;
    const uint32_t r = a.ridx[t];
    // the head's position in the run order (row 0 or key order)
    const uint32_t e0 = a.order ? j : a.links[((size_t)t * D) * 4 + 2].y;
    // the run ends at the next boundary (row-0 order)
    const uint32_t e_end = a.bpos[a.bidx[e0] + 1];
    const uint32_t L = e_end - e0;
    const uint32_t hasdel = a.delpre[e_end] != a.delpre[e0];
    RunRec<D> rec;
    rec.e0 = e0;
    rec.info = L | (hasdel << 31);
    rec.bits0 = 0;
    if (a.dmask) rec.bits0 = a.dmask[j];  // SF1 / CU: the rows this run's ops drop (by key-order position)
    if (a.delbits && hasdel) {
      const uint32_t sh = e0 & 31u;
      uint32_t b = a.delbits[e0 >> 5] >> sh;
      if (sh) b |= a.delbits[(e0 >> 5) + 1] << (32u - sh);
      rec.bits0 = L >= 32 ? b : (b & ((1u << L) - 1u));
    }
    const bool head_del = a.opflags[e0] & 1u;
#pragma unroll
    for (int i = 0; i < D; ++i) {
      // the (t, row) link record, one 256-bit load: {rank, prev, own count,
      // max of the other slots} {cell, sorted position, 0, 0}
      uint4 l0 = make_uint4(0u, 0u, 0u, 0u), l1 = make_uint4(0u, 0u, 0u, 0u);
      if (!((rec.bits0 >> i) & 1u) || !a.dmask) ld_sector(a.links + ((size_t)t * D + i) * 4, l0, l1);
      rec.cells[i] = l1.x;
      rec.rank[i] = l0.x;
      if (a.obs2) {
        rec.A[i] = head_del ? l0.z + 1u : l0.z - 1u;
        rec.O[i] = l0.w;
      } else {
        rec.A[i] = 0;
        rec.O[i] = 0;
      }
    }
    {  // whole sectors (streaming): read back by the engine (prefetched ahead)
      static_assert(sizeof(RunRec<D>) % 32 == 0, "run records are whole sectors");
      const uint4* src = reinterpret_cast<const uint4*>(&rec);
      uint4* dst = reinterpret_cast<uint4*>(a.recs + r);
#pragma unroll
      for (int q = 0; q < (int)(sizeof(RunRec<D>) / 32); ++q) st_sector(dst + 2 * q, src[2 * q], src[2 * q + 1]);
    }
  }
}

// ---------------------------------------------------------------- 5. engine
__device__ unsigned long long g_engine_stats[8];
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }

struct RowMap {
  int32_t l, u, p0, pW;
};
struct WalkPiece {
  int32_t S, mx;  // net steps (delete +1 / insert -1) and max prefix (dominance over the piece)
};
constexpr int32_t MAP_INF = 0x3fffffff;
constexpr uint32_t NO_OWNER = 0xFFFFFFFFu;
constexpr int MAP_LEVELS = 3;  // pieces of 1, 32 and 1024 words

template <int D>
struct EngineArgs {
  unsigned long long* slim64;  // (seq << 32 | value) per slim cell
  const RunRec<D>* recs;
  const uint32_t* opdata;      // SF1: b_min per op (row-0 order)
  const uint32_t* delbits;     // SFF: delete flags in row-0 order, one bit per op
  const uint32_t* wsum;        // SFF: per aligned word, nd | -min prefix << 6 | max prefix << 12 | draw-up << 18
  const WalkPiece* piece[3];   // SFF long runs: pieces of 1, 32, 1024 aligned words (word_maps_k, block_maps_k)
  const RowMap* rmap[3];       //   and their per-row reflected-walk maps (null: no long-run path)
  Ctl* ctl;
  unsigned long long* inc;     // int64[d] tallies (two's complement add)
  uint32_t budget;             // ops a lane replays per engine iteration before it yields
  int b_opdata;                // MODE 3: an insert's b_min comes from opdata (SF2) instead of A0 + x
  const uint32_t* omax[2];     // insert-only per-op caps (CML, oracle-assisted): max cap per 32 / 1024 ops
  const uint32_t* brk_pre;     // oracle-assisted: exclusive prefix count of ops whose cap does not exceed the previous op's
  unsigned long long* trace;   // diagnostics: per run {claim, ready, done} globaltimer ns (or null)
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}



// Replay position inside the run a lane executes (SFF runs may span several
// engine iterations).
struct Cursor {
  uint32_t m, x, e, rem, A0;
  uint32_t blk;      // 128-op block (4 words) held in q0
  uint4 q0, q1, q2;  // delete-bit prefetch: up to 12 words ahead of the replay
  bool ring;
};

__device__ __forceinline__ uint32_t pick_word(const uint4& q, uint32_t sel) {
  return sel == 0 ? q.x : sel == 1 ? q.y : sel == 2 ? q.z : q.w;
}

template <int D>
__device__ __forceinline__ void raise_to(uint32_t tgt, uint32_t (&c)[D], uint32_t (&raised)[D]) {
#pragma unroll
  for (int i = 0; i < D; ++i)
    if (c[i] < tgt) { raised[i] += tgt - c[i]; c[i] = tgt; }
}

// Walk summaries of +1 (delete) / -1 (insert) step sequences. For a byte b
// (8 steps, bit j = step j) lut[b] packs, each biased by +8 into one byte:
// the total, the minimum and maximum prefix sums (empty prefix included) and
// the maximum draw-up (largest rise between two prefixes).
struct WalkSum {
  int32_t t, mn, mx, du;
};

__device__ __forceinline__ void build_step_lut(uint32_t* lut) {
  for (uint32_t b = threadIdx.x; b < 256; b += blockDim.x) {
    int32_t p = 0, mn = 0, mx = 0, du = 0;
    for (int j = 0; j < 8; ++j) {
      p += ((b >> j) & 1u) ? 1 : -1;
      mn = min(mn, p);
      mx = max(mx, p);
      du = max(du, p - mn);
    }
    lut[b] = (uint32_t)(p + 8) | ((uint32_t)(mn + 8) << 8) | ((uint32_t)(mx + 8) << 16) | ((uint32_t)(du + 8) << 24);
  }
}

// Two-sided reflection tables for narrow rows: for an upper bound W in
// [1, WMAX], a start v in [0, 7] and a byte of steps b, rlut[((W-1)*8+v)*256+b]
// = (pushes at the lower bound << 4) | end value, where an insert maps
// v -> max(v-1, 0) (v == 0 is a push) and a delete v -> min(v+1, W).
constexpr int WMAX = 7;

__device__ __forceinline__ void build_reflect_lut(uint8_t* rlut) {
  for (uint32_t idx = threadIdx.x; idx < (uint32_t)WMAX * 8 * 256; idx += blockDim.x) {
    const uint32_t b = idx & 255u, v0 = (idx >> 8) & 7u, W = (idx >> 11) + 1u;
    uint32_t v = v0, push = 0;
    for (int j = 0; j < 8; ++j) {
      if ((b >> j) & 1u) {
        v = min(v + 1u, W);
      } else if (v == 0) {
        ++push;
      } else {
        --v;
      }
    }
    rlut[idx] = (uint8_t)((push << 4) | v);
  }
}

// summary of a full 32-step word: fold the four byte summaries
__device__ __forceinline__ WalkSum walk_sum32(uint32_t bits, const uint32_t* lut) {
  WalkSum w{0, 0, 0, 0};
#pragma unroll
  for (int byte = 0; byte < 4; ++byte) {
    const uint32_t e = lut[(bits >> (8 * byte)) & 0xFFu];
    const int32_t t = (int32_t)(e & 0xFFu) - 8, mn = (int32_t)((e >> 8) & 0xFFu) - 8;
    const int32_t mx = (int32_t)((e >> 16) & 0xFFu) - 8, du = (int32_t)(e >> 24) - 8;
    w.du = max(max(w.du, du), w.t + mx - w.mn);
    w.mn = min(w.mn, w.t + mn);
    w.mx = max(w.mx, w.t + mx);
    w.t += t;
  }
  return w;
}

// per-word walk summaries of the delete bits (for the steady fast loop)
__global__ void __launch_bounds__(256) word_sums_k(const uint32_t* __restrict__ delbits, uint32_t nwords,
                                                   uint32_t* __restrict__ wsum) {
  __shared__ uint32_t lut[256];
  build_step_lut(lut);
  __syncthreads();
  for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < nwords; w += gridDim.x * blockDim.x) {
    const uint32_t bits = delbits[w];
    const WalkSum s = walk_sum32(bits, lut);
    wsum[w] = (uint32_t)__popc(bits) | ((uint32_t)(-s.mn) << 6) | ((uint32_t)s.mx << 12) | ((uint32_t)s.du << 18);
  }
}

// ---- reflected-walk maps for long SFF runs ----------------------------------
// Inside a run in the steady regime (m == A0 + x) with the key's own slot
// dominating its buckets (O_i <= A_i + x), every row evolves on its own as a
// two-sided reflected walk v -> [0, W_i] (v_i = c_i - A0 - x, W_i = A_i - A0):
// an insert maps v -> max(v - 1, 0) (a push at 0 is one raise), a delete
// v -> min(v + 1, W_i). Any stretch of such steps acts on [0, W] as
// h(v) = min(max(v + S, l), u) and raises p(v) = pW + max(p0 - pW - v, 0)
// times (coupling: paths from v and v + 1 stay one apart until the lower one
// is pushed or the upper one capped; lower pushes come first for small v).
// Both compose in O(1), so the engine finishes a long run by applying a few
// precomputed pieces (32-op words, 1024-op and 32768-op blocks) instead of
// replaying it op by op.

__device__ __forceinline__ int32_t rowmap_apply(const RowMap& f, int32_t S, int32_t v) {
  return min(max(v + S, f.l), f.u);
}
__device__ __forceinline__ int32_t rowmap_push(const RowMap& f, int32_t v) {
  return f.pW + max(f.p0 - f.pW - v, 0);
}
// f (net S1) followed by g (net S2), on [0, W]
__device__ __forceinline__ RowMap rowmap_cat(const RowMap& f, int32_t S1, const RowMap& g, int32_t S2, int32_t W) {
  RowMap h;
  int32_t L = max(f.l + S2, g.l);
  int32_t U = min(max(f.u + S2, g.l), g.u);
  if (L > U) L = U;
  h.l = max(L, -MAP_INF);
  h.u = min(U, MAP_INF);
  h.p0 = f.p0 + rowmap_push(g, rowmap_apply(f, S1, 0));
  h.pW = f.pW + rowmap_push(g, rowmap_apply(f, S1, W));
  return h;
}

// the upper bound of row i's reflected walk: W_i = A_i - A0 for the SFF max
// clamp; K_i = A_i - A0 + O_i for the SF3/SF4 sum trigger (O_i = the other
// slots' sum), whose rows step v -> v + [v < K_i] on a delete
template <int D>
__device__ __forceinline__ int32_t walk_width(const RunRec<D>& rec, int i, uint32_t A0, int sum_mode) {
  const uint64_t wd = (uint64_t)(rec.A[i] - A0) + (sum_mode ? (uint64_t)rec.O[i] : 0ull);
  return (int32_t)min(wd, (uint64_t)MAP_INF);
}

// owner of every aligned word of a long SFF run (hasdel, L > 32): the run id
template <int D>
__global__ void __launch_bounds__(256) long_owner_k(const RunRec<D>* __restrict__ recs, const Ctl* __restrict__ ctl,
                                                    uint32_t* __restrict__ wowner) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t R = ctl->n_runs;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t base = warp * 32u; base < R; base += nwarps * 32u) {
    const uint32_t r = base + lane;
    uint32_t wa = 1, wl = 0;
    if (r < R) {
      const uint32_t e0 = recs[r].e0, info = recs[r].info, L = info & 0x7fffffffu;
      if ((info >> 31) && L > 32u) wa = (e0 + 31u) >> 5, wl = (e0 + L - 1u) >> 5;
    }
    unsigned todo = __ballot_sync(0xffffffffu, wa <= wl);
    while (todo) {
      const int src = __ffs(todo) - 1;
      todo &= todo - 1u;
      const uint32_t a0 = __shfl_sync(0xffffffffu, wa, src), a1 = __shfl_sync(0xffffffffu, wl, src);
      const uint32_t rr = base + (uint32_t)src;
      for (uint32_t w = a0 + lane; w <= a1; w += 32u) wowner[w] = rr;
    }
  }
}

// validated owner of word w (stale entries from earlier calls never match)
template <int D>
__device__ __forceinline__ uint32_t word_owner(const uint32_t* wowner, const RunRec<D>* recs, uint32_t R, uint32_t w,
                                               uint32_t& e0, uint32_t& L) {
  const uint32_t r = wowner[w];
  if (r >= R) return NO_OWNER;
  e0 = recs[r].e0;
  const uint32_t info = recs[r].info;
  L = info & 0x7fffffffu;
  if (!(info >> 31) || L <= 32u) return NO_OWNER;
  if (w < ((e0 + 31u) >> 5) || w > ((e0 + L - 1u) >> 5)) return NO_OWNER;
  return r;
}

// level 0: one piece per aligned word of a long run (the run's last word
// masked to its end), every row with its own W_i
template <int D>
__global__ void __launch_bounds__(256) word_maps_k(const RunRec<D>* __restrict__ recs, const Ctl* __restrict__ ctl,
                                                   const uint32_t* __restrict__ wowner,
                                                   const uint32_t* __restrict__ delbits, uint32_t nwords,
                                                   WalkPiece* __restrict__ piece, RowMap* __restrict__ rmap,
                                                   int sum_mode) {
  const uint32_t R = ctl->n_runs;
  for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < nwords; w += gridDim.x * blockDim.x) {
    uint32_t e0, L;
    const uint32_t r = word_owner<D>(wowner, recs, R, w, e0, L);
    if (r == NO_OWNER) continue;
    const uint32_t cnt = min(e0 + L - w * 32u, 32u);
    const uint32_t bits = delbits[w] & (cnt == 32u ? 0xFFFFFFFFu : ((1u << cnt) - 1u));
    uint32_t A0 = recs[r].A[0];
#pragma unroll
    for (int i = 1; i < D; ++i) A0 = min(A0, recs[r].A[i]);
    int32_t S = 0, mx = 0;
    for (uint32_t j = 0; j < cnt; ++j) {
      S += ((bits >> j) & 1u) ? 1 : -1;
      mx = max(mx, S);
    }
    piece[w] = WalkPiece{S, mx};
#pragma unroll
    for (int i = 0; i < D; ++i) {
      const int32_t W = walk_width<D>(recs[r], i, A0, sum_mode);
      int32_t l = -MAP_INF, u = MAP_INF, s = 0, v0 = 0, vW = W, p0 = 0, pW = 0;
      for (uint32_t j = 0; j < cnt; ++j) {
        if ((bits >> j) & 1u) {  // delete: (a = +1, l = -inf, u = W)
          l = l + 1;
          u = min(u + 1, W);
          if (l > u) l = u;
          ++s;
          v0 = min(v0 + 1, W);
          vW = min(vW + 1, W);
        } else {  // insert: (a = -1, l = 0, u = inf)
          l = max(l - 1, 0);
          u = max(u - 1, 0);
          --s;
          p0 += v0 == 0;
          pW += vW == 0;
          v0 = max(v0 - 1, 0);
          vW = max(vW - 1, 0);
        }
      }
      rmap[(size_t)w * D + i] = RowMap{max(l, -MAP_INF), min(u, MAP_INF), p0, pW};
    }
  }
}

// level k > 0: piece b composes 32 consecutive level-(k-1) pieces when its
// 32^k words all belong to one long run
template <int D>
__global__ void __launch_bounds__(256) block_maps_k(const RunRec<D>* __restrict__ recs, const Ctl* __restrict__ ctl,
                                                    const uint32_t* __restrict__ wowner, uint32_t nwords,
                                                    uint32_t span, const WalkPiece* __restrict__ pin,
                                                    const RowMap* __restrict__ rin, WalkPiece* __restrict__ pout,
                                                    RowMap* __restrict__ rout, uint32_t nblocks, int sum_mode) {
  const uint32_t R = ctl->n_runs;
  for (uint32_t bk = blockIdx.x * blockDim.x + threadIdx.x; bk < nblocks; bk += gridDim.x * blockDim.x) {
    const uint32_t w0 = bk * span, w1 = w0 + span - 1u;
    if (w1 >= nwords) continue;
    uint32_t e0, L, e0b, Lb;
    const uint32_t r = word_owner<D>(wowner, recs, R, w0, e0, L);
    if (r == NO_OWNER || word_owner<D>(wowner, recs, R, w1, e0b, Lb) != r) continue;
    uint32_t A0 = recs[r].A[0];
#pragma unroll
    for (int i = 1; i < D; ++i) A0 = min(A0, recs[r].A[i]);
    int32_t W[D];
    RowMap acc[D];
    WalkPiece pc = pin[bk * 32u];
#pragma unroll
    for (int i = 0; i < D; ++i) {
      W[i] = walk_width<D>(recs[r], i, A0, sum_mode);
      acc[i] = rin[(size_t)(bk * 32u) * D + i];
    }
    for (uint32_t q = 1; q < 32u; ++q) {
      const WalkPiece nx = pin[bk * 32u + q];
#pragma unroll
      for (int i = 0; i < D; ++i) acc[i] = rowmap_cat(acc[i], pc.S, rin[(size_t)(bk * 32u + q) * D + i], nx.S, W[i]);
      pc.mx = max(pc.mx, pc.S + nx.mx);
      pc.S += nx.S;
    }
    pout[bk] = pc;
#pragma unroll
    for (int i = 0; i < D; ++i) rout[(size_t)bk * D + i] = acc[i];
  }
}

// SFF: replay `avail` ops of a run whose delete flags are the low bits of
// `bits`. Within a run no other op touches the key's d buckets, so in row i
// the key's own slot count is A_i + x (x = the run's net inserts so far) and
// the other slots keep their maximum O_i: an insert's b_min is min_i A_i + x
// and a delete clamps row i to max(A_i + x, O_i).
template <int D>
__device__ __forceinline__ void replay_word(uint32_t bits, uint32_t avail, const uint32_t (&A)[D],
                                            const uint32_t (&O)[D], uint32_t A0, uint32_t& m, uint32_t& x,
                                            uint32_t (&c)[D], uint32_t (&raised)[D], uint32_t (&ws)[5],
                                            const uint32_t* lut, const uint8_t* rlut) {
  const uint32_t nd = __popc(bits), ni = avail - nd;
  // Gap word: the min lags the key's own count by at least the word's
  // deletes (mu = m - x, mu + nd <= A0). Every insert passes the gate and
  // deletes only shrink caps that stay above every row (c_i + nd <= A_i + x),
  // so a row's offset v = c_i - m drops by one per insert down to 0, each
  // insert at v = 0 being one raise.
  {
    bool gap = (uint64_t)m + nd <= (uint64_t)(uint32_t)(A0 + x);
#pragma unroll
    for (int i = 0; i < D; ++i)
      gap = gap && (int64_t)O[i] <= (int64_t)(uint32_t)(A[i] + x) - (int64_t)nd &&
            (uint64_t)c[i] + nd <= (uint64_t)(uint32_t)(A[i] + x);
    if (gap) {
#pragma unroll
      for (int i = 0; i < D; ++i) {
        const uint32_t v = c[i] - m;
        raised[i] += ni > v ? ni - v : 0u;
        c[i] = m + ni + (v > ni ? v - ni : 0u);
      }
      m += ni;
      x += ni - nd;
      ++ws[0];
      return;
    }
  }
  // Steady word: the min is caught up (m == A0 + x, so it stays A0 + x) and
  // no other slot can exceed the key's own count within the word. Rows then
  // evolve independently: with v_i = c_i - m an insert maps v -> max(v-1, 0)
  // (a push at 0 is one raise) and a delete v -> min(v+1, W_i), W_i = A_i -
  // A0. The lower-reflected walk peaks at max(v + max prefix, max draw-up);
  // while that stays <= W_i the upper bound never binds and
  // v_end = max(v + S, S - min prefix) (Lindley), pushes = v_end - (v + S).
  // W_i == 0 pins the row to the min; otherwise the row steps bit by bit.
  {
    bool steady = m == A0 + x;
#pragma unroll
    for (int i = 0; i < D; ++i) steady = steady && (int64_t)O[i] <= (int64_t)(uint32_t)(A[i] + x) - (int64_t)nd;
    if (steady) {
      const int32_t S = (int32_t)nd - (int32_t)ni;
      const uint32_t mnew = m + ni - nd;
      uint32_t v[D], W[D], push[D];
      bool done[D];
#pragma unroll
      for (int i = 0; i < D; ++i) {
        v[i] = c[i] - m;
        W[i] = A[i] - A0;
        push[i] = 0;
        done[i] = false;
      }
      if (avail == 32u) {
        const WalkSum w = walk_sum32(bits, lut);
#pragma unroll
        for (int i = 0; i < D; ++i) {
          if ((int64_t)max((int64_t)v[i] + w.mx, (int64_t)w.du) <= (int64_t)W[i]) {  // Lindley
            const int64_t vend = max((int64_t)v[i] + S, (int64_t)(S - w.mn));
            push[i] = (uint32_t)(vend - ((int64_t)v[i] + S));
            v[i] = (uint32_t)vend;
            done[i] = true;
          } else if (W[i] == 0 && v[i] == 0) {  // the row sits on both bounds
            push[i] = ni;
            done[i] = true;
          }
        }
        // narrow rows: four table steps each, the d chains interleaved
#pragma unroll
        for (int byte = 0; byte < 4; ++byte) {
          const uint32_t b = (bits >> (8 * byte)) & 0xFFu;
#pragma unroll
          for (int i = 0; i < D; ++i) {
            if (!done[i] && W[i] <= (uint32_t)WMAX && W[i] > 0 && v[i] <= 7u) {
              const uint32_t e = rlut[((W[i] - 1u) * 8u + v[i]) * 256u + b];
              push[i] += e >> 4;
              v[i] = e & 15u;
            }
          }
        }
#pragma unroll
        for (int i = 0; i < D; ++i)
          if (!done[i] && W[i] <= (uint32_t)WMAX && W[i] > 0 && v[i] <= 7u) done[i] = true;
      }
#pragma unroll
      for (int i = 0; i < D; ++i) {
        if (!done[i]) {
          if (W[i] == 0 && v[i] == 0) {
            push[i] = ni;
          } else {
            for (uint32_t k = 0; k < avail; ++k) {
              const uint32_t del = (bits >> k) & 1u;
              push[i] += (del == 0u) & (v[i] == 0u);
              v[i] = del ? min(v[i] + 1u, W[i]) : (v[i] ? v[i] - 1u : 0u);
            }
          }
        }
        raised[i] += push[i];
        c[i] = mnew + v[i];
      }
      m = mnew;
      x += ni - nd;
      ++ws[1];
      return;
    }
  }
  // general word: op by op, insert stretches in closed form (b_min rises by
  // exactly one per insert, so once one raises all later ones do)
  ++ws[2];
  uint32_t pos = 0;
  while (pos < avail) {
    const uint32_t rest = bits >> pos;
    const uint32_t s = min(rest ? (uint32_t)(__ffs(rest) - 1) : 32u, avail - pos);
    if (s) {
      const int64_t diff = (int64_t)m - (int64_t)(uint32_t)(A0 + x);
      const int64_t kstar = diff + 1 > 1 ? diff + 1 : 1;
      if (kstar <= (int64_t)s) {
        m += (uint32_t)((int64_t)s - kstar + 1);
        raise_to<D>(m, c, raised);
      }
      x += s;
      pos += s;
    }
    if (pos < avail) {  // a delete
      x -= 1u;
      m = U32MAX;
#pragma unroll
      for (int i = 0; i < D; ++i) {
        c[i] = min(c[i], max(A[i] + x, O[i]));
        m = min(m, c[i]);
      }
      pos += 1;
    }
  }
}

// Advance the run a lane executes; true once it is complete.
// MODE 0: SF1 (insert-only runs; b_min strictly increases along a same-key
//         run, so the first op with b_k > m0 raises and so does every later)
// MODE 1: CU (every insert raises; saturation ruled out by the host precheck)
// MODE 2: SFF (see replay_word)
// MODE 3: SF2 / SF3 / SF4 (a delete decrements each row whose slim counter
//         exceeds that row's observation: the bucket / fold-group sum, or the
//         deletion sub-sketch counter; A_i + x + O_i within the run)
template <int D, int MODE>
__device__ __forceinline__ bool replay_step(const EngineArgs<D>& a, Cursor& k, uint32_t e0, uint32_t info,
                                            uint32_t bits0, const uint32_t (&A)[D], const uint32_t (&O)[D],
                                            uint32_t (&c)[D], uint32_t (&raised)[D], uint32_t (&ws)[5],
                                            const uint32_t* lut, const uint8_t* rlut) {
  const uint32_t L = info & 0x7fffffffu;
  if (MODE == 1) {
    raise_to<D>(k.m + L, c, raised);  // m0 + L fits: the precheck bounds every counter
    return true;
  }
  if (MODE == 0) {
    // b_min strictly increases along a same-key SF1 run (the key's own fat
    // cells gain one per op): the first raising op by binary search
    uint32_t j = 0, hi = L;
    while (j < hi) {
      const uint32_t mid = (j + hi) >> 1;
      if (a.opdata[e0 + mid] <= k.m) j = mid + 1; else hi = mid;
    }
    if (L - j) raise_to<D>(k.m + (L - j), c, raised);
    return true;
  }
  if (MODE == 3) {
    // insert-only SF3/SF4 run: b_min = A0 + j, closed form as SFF. (SF2's
    // b_min comes from the flat fat, where other keys' deletes may lower it
    // mid-run, so SF2 runs always replay op by op.)
    if (!(info >> 31) && !a.b_opdata) {
      const int64_t jstar = max((int64_t)k.m - (int64_t)k.A0 + 1, (int64_t)1);
      if (jstar <= (int64_t)L) raise_to<D>(k.m + (uint32_t)((int64_t)L - jstar + 1), c, raised);
      return true;
    }
    // op by op, one delete-bit word at a time; at aligned words of a long
    // run with every row in [0, K_i] (c_i >= A0 + x: not lagging), rows are
    // independent two-sided reflected walks and precomputed pieces apply
    uint32_t budget = a.budget;
    if (a.brk_pre && k.rem == L && (L == 1 || a.brk_pre[e0 + L] == a.brk_pre[e0 + 1])) {
      // caps strictly increase along the run (exact true counts of one key):
      // once an op raises, every later op does (its cap exceeds the new
      // minimum), so the first raising op by binary search, as SF1
      uint32_t j = 0, hi = L;
      while (j < hi) {
        const uint32_t mid = (j + hi) >> 1;
        if (a.opdata[e0 + mid] <= k.m) j = mid + 1; else hi = mid;
      }
      if (L - j) raise_to<D>(k.m + (L - j), c, raised);
      k.x += L;
      k.e += L;
      k.rem = 0;
      return true;
    }
    while (k.rem && budget) {
      if (a.omax[0]) {
        // insert-only caps: an op raises only if m < its cap, so aligned
        // blocks (1024 ops) and words (32 ops) whose largest cap is <= m
        // change nothing but the insert count; skip them whole
        const uint32_t* o0 = a.omax[0];
        const uint32_t* o1 = a.omax[1];
        while (k.rem && budget) {
          if ((k.e & 1023u) == 0 && k.rem >= 1024u && __ldg(o1 + (k.e >> 10)) <= k.m) {
            k.e += 1024u, k.rem -= 1024u, k.x += 1024u, budget -= min(budget, 32u), ++ws[3];
            continue;
          }
          const uint32_t av = min(32u - (k.e & 31u), k.rem);
          if (__ldg(o0 + (k.e >> 5)) <= k.m) {
            k.e += av, k.rem -= av, k.x += av, budget -= min(budget, 8u), ++ws[3];
            continue;
          }
          break;
        }
        if (!k.rem || !budget) break;
      }
      if (!a.b_opdata && a.rmap[0] && L > 32u && (k.e & 31u) == 0) {
        const int64_t floor0 = (int64_t)(uint32_t)(k.A0 + k.x);
        int32_t v[D];
        bool ok = true;
#pragma unroll
        for (int i = 0; i < D; ++i) {
          const int64_t vi = (int64_t)c[i] - floor0;
          const int64_t Ki = (int64_t)(A[i] - k.A0) + (int64_t)O[i];
          ok = ok && vi >= 0 && vi <= Ki && Ki < (int64_t)MAP_INF;
          v[i] = (int32_t)vi;
        }
        if (ok) {
          const uint32_t end = e0 + L, wl = (end - 1u) >> 5;
          uint32_t w = k.e >> 5;
          int64_t x = (int64_t)(int32_t)k.x;
          while (w <= wl) {
            int lvl = 0;
            if ((w & 1023u) == 0 && w + 1023u <= wl) lvl = 2;
            else if ((w & 31u) == 0 && w + 31u <= wl) lvl = 1;
            const uint32_t idx = w >> (5 * lvl);
            const WalkPiece* pp = lvl == 2 ? a.piece[2] : lvl == 1 ? a.piece[1] : a.piece[0];
            const RowMap* rp = lvl == 2 ? a.rmap[2] : lvl == 1 ? a.rmap[1] : a.rmap[0];
            const WalkPiece pc = pp[idx];
#pragma unroll
            for (int i = 0; i < D; ++i) {
              const RowMap f = rp[(size_t)idx * D + i];
              raised[i] += (uint32_t)rowmap_push(f, v[i]);
              v[i] = rowmap_apply(f, pc.S, v[i]);
            }
            x -= pc.S;
            w += 1u << (5 * lvl);
            ++ws[3];
          }
          const uint32_t ne = end;
          ws[4] += ne - k.e;
          k.x = (uint32_t)(int32_t)x;
          uint32_t m = U32MAX;
#pragma unroll
          for (int i = 0; i < D; ++i) {
            c[i] = k.A0 + k.x + (uint32_t)v[i];
            m = min(m, c[i]);
          }
          k.m = m;
          k.rem = 0;
          k.e = ne;
          break;
        }
      }
      if (a.b_opdata && (k.e & 31u) == 0 && k.rem >= 64u && budget >= 64u) {
        // whole words of a long run with per-op caps: the next words' caps
        // and delete bits are prefetched into L1 while this word replays
        uint32_t w = k.e >> 5;
        const uint32_t nwf = min(k.rem, budget) >> 5;
        const uint4* src = reinterpret_cast<const uint4*>(a.opdata);
        for (uint32_t wi = 0; wi < nwf; ++wi, ++w) {
          if (wi + 2 < nwf) {
            asm volatile("prefetch.global.L1 [%0];" ::"l"(src + (size_t)(w + 2) * 8));
            if (((w + 2) & 31u) == 0) asm volatile("prefetch.global.L1 [%0];" ::"l"(a.delbits + w + 2));
          }
          uint4 cb[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) cb[q] = __ldg(src + (size_t)w * 8 + q);
          const uint32_t cdb = __ldg(a.delbits + w);
          {
            // collapsed replay: while no delete binds, every row is
            // max(its value at the word start, m), so only the scalar min
            // moves (m += [m < cap] per insert); a delete must keep every
            // row <= A_i + O_i + x. If one would bind, redo the word exactly.
            int64_t capmin = INT64_MAX, cmc = INT64_MIN;
#pragma unroll
            for (int i = 0; i < D; ++i) {
              const int64_t cap = (int64_t)A[i] + (int64_t)O[i];
              capmin = min(capmin, cap);
              cmc = max(cmc, (int64_t)c[i] - cap);
            }
            uint32_t mm = k.m;
            int32_t xx = (int32_t)k.x;
            bool okc = true;
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) {
              const uint4 v4 = cb[jj >> 2];
              const uint32_t ob = (jj & 3) == 0 ? v4.x : (jj & 3) == 1 ? v4.y : (jj & 3) == 2 ? v4.z : v4.w;
              if (!((cdb >> jj) & 1u)) {
                xx += 1;
                mm += mm < ob ? 1u : 0u;
              } else {
                xx -= 1;
                okc = okc && (int64_t)mm - capmin <= (int64_t)xx && cmc <= (int64_t)xx;
              }
            }
            if (okc) {
#pragma unroll
              for (int i = 0; i < D; ++i) {
                const uint32_t nc = max(c[i], mm);
                raised[i] += nc - c[i];
                c[i] = nc;
              }
              k.m = mm;
              k.x = (uint32_t)xx;
              ++ws[3];
              continue;
            }
          }
          {
            // exact replay, branch-light 32-bit form: a delete's cap
            // A_i + O_i + x is a count (0 .. 2^32 - 1), so modular u32 math is exact
            uint32_t T[D];
#pragma unroll
            for (int i = 0; i < D; ++i) T[i] = A[i] + O[i];
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) {
              const uint4 v4 = cb[jj >> 2];
              const uint32_t ob = (jj & 3) == 0 ? v4.x : (jj & 3) == 1 ? v4.y : (jj & 3) == 2 ? v4.z : v4.w;
              if (!((cdb >> jj) & 1u)) {
                k.x += 1u;
                const uint32_t up = k.m < ob ? 1u : 0u;
#pragma unroll
                for (int i = 0; i < D; ++i) {
                  const uint32_t r = (c[i] == k.m) ? up : 0u;
                  c[i] += r;
                  raised[i] += r;
                }
                k.m += up;
              } else {
                k.x -= 1u;
                uint32_t m = U32MAX;
#pragma unroll
                for (int i = 0; i < D; ++i) {
                  c[i] -= c[i] > T[i] + k.x ? 1u : 0u;
                  m = min(m, c[i]);
                }
                k.m = m;
              }
            }
          }
        }
        k.e += nwf * 32u;
        k.rem -= nwf * 32u;
        budget -= nwf * 32u;
        ws[2] += nwf;
        continue;
      }
      const uint32_t off = k.e & 31u, avail = min(min(32u - off, k.rem), budget);
      const uint32_t bits = a.delbits[k.e >> 5] >> off;
      if (a.b_opdata) {
        // SF2: the word's 32 b_min values in one batch of 16-B loads (one
        // memory latency per word instead of one per insert), then the ops
        // with static register indices
        uint32_t ob[32];
        const uint4* src = reinterpret_cast<const uint4*>(a.opdata + (k.e & ~31u));
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const uint4 v = __ldg(src + q);
          ob[4 * q] = v.x; ob[4 * q + 1] = v.y; ob[4 * q + 2] = v.z; ob[4 * q + 3] = v.w;
        }
        const uint32_t wb = bits << off;  // delete bits at their word positions
#pragma unroll
        for (uint32_t jj = 0; jj < 32u; ++jj) {
          if (jj < off || jj >= off + avail) continue;
          if (!((wb >> jj) & 1u)) {
            k.x += 1u;
            if (k.m < ob[jj]) {
#pragma unroll
              for (int i = 0; i < D; ++i)
                if (c[i] == k.m) c[i] += 1u, raised[i] += 1u;
              k.m += 1u;
            }
          } else {
            k.x -= 1u;
            uint32_t m = U32MAX;
#pragma unroll
            for (int i = 0; i < D; ++i) {
              const int64_t T = (int64_t)A[i] + (int64_t)(int32_t)k.x + (int64_t)O[i];
              if ((int64_t)c[i] > T) c[i] -= 1u;
              m = min(m, c[i]);
            }
            k.m = m;
          }
        }
        k.e += avail;
        k.rem -= avail;
        budget -= avail;
        ws[2] += 1;
        continue;
      }
      for (uint32_t j = 0; j < avail; ++j) {
        if (!((bits >> j) & 1u)) {  // insert
          k.x += 1u;
          const uint32_t b = k.A0 + k.x;
          if (k.m < b) {
#pragma unroll
            for (int i = 0; i < D; ++i)
              if (c[i] == k.m) c[i] += 1u, raised[i] += 1u;
            k.m += 1u;
          }
        } else {  // delete
          k.x -= 1u;
          uint32_t m = U32MAX;
#pragma unroll
          for (int i = 0; i < D; ++i) {
            const int64_t T = (int64_t)A[i] + (int64_t)(int32_t)k.x + (int64_t)O[i];
            if ((int64_t)c[i] > T) c[i] -= 1u;
            m = min(m, c[i]);
          }
          k.m = m;
        }
      }
      k.e += avail;
      k.rem -= avail;
      budget -= avail;
      ws[2] += 1;
    }
    return k.rem == 0;
  }
  if (SHORT_RUNS && (info >> 31) && L <= SHORT_RUN_MAX && k.rem == L) {
    // short run (its delete bits are all in bits0): op by op
    // with the same few instructions in every lane, so a warp's lanes that
    // became ready together replay in lockstep instead of serialising the
    // word-replay paths. Insert: own counts A_i + x, gate m < A0 + x, raise
    // the rows at m. Delete: c_i = min(c_i, max(A_i + x, O_i)).
    uint32_t m = k.m, x = k.x;
    for (uint32_t j = 0; j < L; ++j) {
      if (!((bits0 >> j) & 1u)) {
        x += 1u;
        if (m < k.A0 + x) {
#pragma unroll
          for (int i = 0; i < D; ++i)
            if (c[i] == m) c[i] += 1u, raised[i] += 1u;
          m += 1u;
        }
      } else {
        x -= 1u;
        m = U32MAX;
#pragma unroll
        for (int i = 0; i < D; ++i) {
          c[i] = min(c[i], max(A[i] + x, O[i]));
          m = min(m, c[i]);
        }
      }
    }
    k.m = m;
    k.x = x;
    k.e += L;
    k.rem = 0;
    return true;
  }
  if (!(info >> 31)) {  // insert-only SFF run: the j-th insert raises iff m0 < A0 + j
    const int64_t jstar = max((int64_t)k.m - (int64_t)k.A0 + 1, (int64_t)1);
    if (jstar <= (int64_t)L) raise_to<D>(k.m + (uint32_t)((int64_t)L - jstar + 1), c, raised);
    return true;
  }
  const uint32_t wlast = (e0 + L - 1) >> 5;
  uint32_t budget = a.budget;
  // steady-word fast loop constants: rows' widths and the largest O_i - A_i
  uint32_t W[D];
  int64_t omax = INT64_MIN;
#pragma unroll
  for (int i = 0; i < D; ++i) {
    W[i] = A[i] - k.A0;
    omax = max(omax, (int64_t)O[i] - (int64_t)A[i]);
  }
  while (k.rem && budget) {
    // Long-run path: at an aligned word in the steady regime with every row
    // inside [0, W_i], apply precomputed reflected-walk pieces (1, 32 or
    // 1024 words) while the key's own slot keeps dominating its buckets.
    if (a.rmap[0] && L > 32u && (k.e & 31u) == 0 && k.m == k.A0 + k.x) {
      int32_t v[D];
      bool ok = true;
      int64_t omax = INT64_MIN;
#pragma unroll
      for (int i = 0; i < D; ++i) {
        const uint32_t vi = c[i] - k.m, Wi = A[i] - k.A0;
        ok = ok && vi <= Wi && Wi < (uint32_t)MAP_INF;
        v[i] = (int32_t)vi;
        omax = max(omax, (int64_t)O[i] - (int64_t)A[i]);
      }
      if (ok) {
        const uint32_t end = e0 + L, wl = (end - 1u) >> 5;
        uint32_t w = k.e >> 5;
        int64_t x = (int64_t)(int32_t)k.x;
        while (w <= wl) {
          int lvl = 0;
          if ((w & 1023u) == 0 && w + 1023u <= wl) lvl = 2;
          else if ((w & 31u) == 0 && w + 31u <= wl) lvl = 1;
          const uint32_t idx = w >> (5 * lvl);
          // (selects, not a dynamic index into the kernel parameters)
          const WalkPiece* pp = lvl == 2 ? a.piece[2] : lvl == 1 ? a.piece[1] : a.piece[0];
          const RowMap* rp = lvl == 2 ? a.rmap[2] : lvl == 1 ? a.rmap[1] : a.rmap[0];
          const WalkPiece pc = pp[idx];
          if (omax > x - pc.mx) break;  // the own slot may stop dominating inside this piece
#pragma unroll
          for (int i = 0; i < D; ++i) {
            const RowMap f = rp[(size_t)idx * D + i];
            raised[i] += (uint32_t)rowmap_push(f, v[i]);
            v[i] = rowmap_apply(f, pc.S, v[i]);
          }
          x -= pc.S;
          w += 1u << (5 * lvl);
          ++ws[3];
        }
        const uint32_t ne = min(w * 32u, end);
        ws[4] += ne - k.e;
        if (ne != k.e) {
          k.x = (uint32_t)(int32_t)x;
          k.m = k.A0 + k.x;
#pragma unroll
          for (int i = 0; i < D; ++i) c[i] = k.m + (uint32_t)v[i];
          k.rem -= ne - k.e;
          k.e = ne;
          if (!k.rem) break;
        }
      }
    }
    // Fast loop over whole aligned words in the steady regime (see
    // replay_word) from the precomputed walk summaries: per word only the
    // regime test and d Lindley updates remain on the sequential path.
    bool fast = (k.e & 31u) == 0 && k.rem >= 32u && budget >= 32u && k.m == k.A0 + k.x;
#pragma unroll
    for (int i = 0; i < D; ++i) fast = fast && W[i] < (1u << 30) && c[i] - k.m < (1u << 30);
    if (fast) {
      // Steady fast loop (32-bit, branch-free per row). m == A0 + x holds by
      // construction inside the loop, so only the O bound and each row's
      // "upper bound out of reach" test remain per word.
      const uint4* ws4 = reinterpret_cast<const uint4*>(a.wsum);
      const uint4* db4 = reinterpret_cast<const uint4*>(a.delbits);
      uint32_t w = k.e >> 5;
      uint4 b0 = ws4[w >> 2], b1 = ws4[(w >> 2) + 1], b2 = ws4[(w >> 2) + 2];
      uint4 d0 = db4[w >> 2], d1 = db4[(w >> 2) + 1], d2 = db4[(w >> 2) + 2];
      int32_t v[D], Wi[D];
#pragma unroll
      for (int i = 0; i < D; ++i) {
        v[i] = (int32_t)(c[i] - k.m);
        Wi[i] = (int32_t)W[i];
      }
      const int32_t om = (int32_t)max(min(omax, (int64_t)INT32_MAX), (int64_t)INT32_MIN + 64);
      int32_t x32 = (int32_t)k.x;
      uint32_t words = 0, wmax = min(k.rem, budget) >> 5;
      while (words < wmax) {
        const uint32_t q = pick_word(b0, w & 3u);
        const int32_t nd = (int32_t)(q & 63u), mn = (int32_t)((q >> 6) & 63u);  // mn = -(min prefix)
        const int32_t mx = (int32_t)((q >> 12) & 63u), du = (int32_t)((q >> 18) & 63u);
        if (x32 - nd < om) break;
        bool easy = true;
#pragma unroll
        for (int i = 0; i < D; ++i) easy = easy & (((v[i] | Wi[i]) == 0) | (max(v[i] + mx, du) <= Wi[i]));
        const int32_t S = 2 * nd - 32;
        if (easy) {
#pragma unroll
          for (int i = 0; i < D; ++i) {
            const bool pinned = (v[i] | Wi[i]) == 0;
            const int32_t vend = pinned ? 0 : max(v[i] + S, S + mn);
            raised[i] += (uint32_t)(pinned ? 32 - nd : vend - v[i] - S);
            v[i] = vend;
          }
        } else {
          // some row can reach its upper bound: narrow rows walk the
          // reflection table, anything wider leaves the fast loop
          bool ok = true;
#pragma unroll
          for (int i = 0; i < D; ++i)
            ok = ok & (((v[i] | Wi[i]) == 0) | (max(v[i] + mx, du) <= Wi[i]) | ((Wi[i] <= WMAX) & (v[i] <= 7)));
          if (!ok) break;
          const uint32_t bits = pick_word(d0, w & 3u);
#pragma unroll
          for (int i = 0; i < D; ++i) {
            const bool pinned = (v[i] | Wi[i]) == 0;
            if (!pinned && max(v[i] + mx, du) > Wi[i]) {  // two-sided reflection: four table steps
              uint32_t vv = (uint32_t)v[i], push = 0;
              const uint8_t* tab = rlut + (uint32_t)(Wi[i] - 1) * 8u * 256u;
#pragma unroll
              for (int byte = 0; byte < 4; ++byte) {
                const uint32_t e = tab[vv * 256u + ((bits >> (8 * byte)) & 0xFFu)];
                push += e >> 4;
                vv = e & 15u;
              }
              raised[i] += push;
              v[i] = (int32_t)vv;
            } else {
              const int32_t vend = pinned ? 0 : max(v[i] + S, S + mn);
              raised[i] += (uint32_t)(pinned ? 32 - nd : vend - v[i] - S);
              v[i] = vend;
            }
          }
        }
        x32 += 32 - 2 * nd;
        ++words;
        ++w;
        if ((w & 3u) == 0) {
          b0 = b1;
          b1 = b2;
          b2 = ws4[(w >> 2) + 2];
          d0 = d1;
          d1 = d2;
          d2 = db4[(w >> 2) + 2];
        }
      }
      k.x = (uint32_t)x32;
      k.m = k.A0 + k.x;
#pragma unroll
      for (int i = 0; i < D; ++i) c[i] = k.m + (uint32_t)v[i];
      k.e += words * 32u;
      k.rem -= words * 32u;
      budget -= words * 32u;
      ws[1] += words;
      if (!k.rem || !budget) break;
    }
    uint32_t bits, avail;
    const uint32_t done = k.e - e0;
    if (done < 32u) {
      avail = min(32u - done, k.rem);
      bits = bits0 >> done;
    } else {
      const uint4* blocks = reinterpret_cast<const uint4*>(a.delbits);
      const uint32_t lastblk = wlast >> 2;
      const uint4 zero4 = make_uint4(0u, 0u, 0u, 0u);
      if (!k.ring || (k.e >> 7) > k.blk + 1u) {
        k.blk = k.e >> 7;
        k.q0 = blocks[k.blk];
        k.q1 = k.blk + 1 <= lastblk ? blocks[k.blk + 1] : zero4;
        k.q2 = k.blk + 2 <= lastblk ? blocks[k.blk + 2] : zero4;
        k.ring = true;
      } else if ((k.e >> 7) != k.blk) {  // advance one block, keep two in flight
        k.q0 = k.q1;
        k.q1 = k.q2;
        ++k.blk;
        k.q2 = k.blk + 2 <= lastblk ? blocks[k.blk + 2] : zero4;
      }
      const uint32_t off = k.e & 31u;
      avail = min(32u - off, k.rem);
      bits = pick_word(k.q0, (k.e >> 5) & 3u) >> off;
    }
    if (avail < 32u) bits &= (1u << avail) - 1u;
    replay_word<D>(bits, avail, A, O, k.A0, k.m, k.x, c, raised, ws, lut, rlut);
    k.e += avail;
    k.rem -= avail;
    budget = budget > avail ? budget - avail : 0u;
  }
  return k.rem == 0;
}

// Ordered engine over runs. Each slim cell is one 64-bit word
// (seq << 32 | value); a run whose head has rank r_i in cell i may execute
// once seq_i == r_i in all its cells, and publishes (r_i + L, value) with a
// single store per cell, so one load both signals readiness and delivers the
// value. Lanes claim runs in stream order of their heads (warp-aggregated
// ticket), so the earliest unfinished run is always ready and the engine
// cannot deadlock. A waiting lane polls only its cells that are not ready
// yet (a ready cell stays ready: nobody else writes it before this run); a
// long run is replayed REPLAY_BUDGET ops per iteration.
template <int D, int MODE>
__global__ void __launch_bounds__(SFK_ENGINE_THREADS, 1) poll_engine_k(EngineArgs<D> a) {
  __shared__ uint32_t lut[256];
  __shared__ uint8_t rlut[WMAX * 8 * 256];
  build_step_lut(lut);
  if (MODE == 2) build_reflect_lut(rlut);
  __syncthreads();
  const uint32_t lane = lane_id();
  const uint32_t R = a.ctl->n_runs;
  bool has = false, exhausted = false;
  uint32_t cells[D], rank[D], A[D], O[D], c[D], raised[D];
  uint32_t e0 = 0, info = 0, bits0 = 0, pend = 0;  // pend: bit i = cell i not seen ready yet
  uint32_t sb[SHORT_CAPS];  // per-op caps of a short run (MODE 3 with per-op data), loaded at claim
#pragma unroll
  for (int q = 0; q < SHORT_CAPS; ++q) sb[q] = 0;
  uint32_t rid = 0;
#pragma unroll
  for (int i = 0; i < D; ++i) raised[i] = 0, cells[i] = 0, rank[i] = 0, A[i] = 0, O[i] = 0, c[i] = 0;
  Cursor k{};
  uint32_t idle = 0;
  uint32_t ws[5] = {0, 0, 0, 0, 0};
  unsigned long long st_cyc = 0, st_runs = 0, st_iters = 0;
  uint32_t pool_base = 0, pool_cnt = 0;  // warp-uniform
  while (true) {
    ++st_iters;
    const unsigned need = __ballot_sync(0xffffffffu, !has && !exhausted);
    if (need) {
      // Claim from the warp's pool of consecutive run ids (one atomic per
      // CLAIM_POOL runs); ids are handed out in increasing order, so the
      // earliest unfinished run is always held by a lane or next in a pool.
      const int leader = __ffs(need) - 1;
      const uint32_t kneed = (uint32_t)__popc(need), pos = (uint32_t)__popc(need & lanemask_lt());
      uint32_t r;
      if (pool_cnt >= kneed) {
        r = pool_base + pos;
        pool_base += kneed;
        pool_cnt -= kneed;
      } else {
        uint32_t nb = 0;
        if ((int)lane == leader) nb = atomicAdd(&a.ctl->qhead, CLAIM_POOL);
        nb = __shfl_sync(0xffffffffu, nb, leader);
        r = pos < pool_cnt ? pool_base + pos : nb + (pos - pool_cnt);
        pool_base = nb + (kneed - pool_cnt);
        pool_cnt = CLAIM_POOL - (kneed - pool_cnt);
      }
      if (!has && !exhausted) {
        if (r + CLAIM_PREFETCH < R) {  // pull a record far ahead into L2 (records exceed L2)
          const char* pf = reinterpret_cast<const char*>(a.recs + r + CLAIM_PREFETCH);
          asm volatile("prefetch.global.L2 [%0];" ::"l"(pf));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(pf + sizeof(RunRec<D>) - 1));
        }
        if (r < R) {
          rid = r;
          if (a.trace) a.trace[3ull * r] = gtimer();
          const RunRec<D>& rec = a.recs[r];
          e0 = rec.e0;
          info = rec.info;
          bits0 = rec.bits0;
#pragma unroll
          for (int i = 0; i < D; ++i) {
            cells[i] = rec.cells[i];
            rank[i] = rec.rank[i];
            if (MODE >= 2) A[i] = rec.A[i], O[i] = rec.O[i];
          }
          pend = (1u << D) - 1u;
          if (MODE <= 1) pend &= ~bits0;  // SF1 / CU: rows this run drops
          if (MODE == 3 && a.b_opdata && (info & 0x7fffffffu) <= (uint32_t)SHORT_CAPS) {
            // issue the short run's cap loads now; they land while its cells are polled
            const uint32_t Ls = info & 0x7fffffffu;
#pragma unroll
            for (int q = 0; q < SHORT_CAPS; ++q) sb[q] = (uint32_t)q < Ls ? __ldg(a.opdata + e0 + q) : 0u;
          }
          // a run that drops every row neither reads nor writes the slim (its
          // ops cannot raise): nothing to replay
          has = MODE > 1 || pend != 0;
        } else {
          exhausted = true;
        }
      }
    }
    // no lane holds a run and none can get one (a lane may also be between
    // runs after claiming one that drops every row)
    if (__all_sync(0xffffffffu, !has && exhausted)) break;
    bool progressed = false;
    if (has && pend) {
      unsigned long long wv[D];
#pragma unroll
      for (int i = 0; i < D; ++i)
        if (pend & (1u << i)) wv[i] = ld_relaxed_u64(a.slim64 + cells[i]);
#pragma unroll
      for (int i = 0; i < D; ++i)
        if ((pend & (1u << i)) && (uint32_t)(wv[i] >> 32) == rank[i]) {
          c[i] = (uint32_t)wv[i];
          pend &= ~(1u << i);
        }
      if (!pend) {  // all cells acquired: start the replay
        if (a.trace) a.trace[3ull * rid + 1] = gtimer();
        if (MODE <= 1) {
#pragma unroll
          for (int i = 0; i < D; ++i)
            if ((bits0 >> i) & 1u) c[i] = U32MAX;  // a dropped row: neither the min nor raised
        }
        k.m = c[0];
#pragma unroll
        for (int i = 1; i < D; ++i) k.m = min(k.m, c[i]);
        k.A0 = A[0];
#pragma unroll
        for (int i = 1; i < D; ++i) k.A0 = min(k.A0, A[i]);
        k.x = 0;
        k.e = e0;
        k.rem = info & 0x7fffffffu;
        k.ring = false;
      }
    }
    if (has && !pend) {
      const long long t0 = clock64();
      bool done;
      if (MODE == 3 && a.b_opdata && k.rem == (info & 0x7fffffffu) && k.rem <= (uint32_t)SHORT_CAPS) {
        // short run with per-op caps (SF2 b_min, CML / oracle caps) from
        // registers: insert x += 1, raise the rows at m when m < cap; delete
        // x -= 1, c_i = c_i - 1 where c_i > A_i + x + O_i
        uint32_t m = k.m;
        int32_t x = (int32_t)k.x;
#pragma unroll
        for (int q = 0; q < SHORT_CAPS; ++q) {
          if ((uint32_t)q >= k.rem) break;
          if (!((bits0 >> q) & 1u)) {
            x += 1;
            if (m < sb[q]) {
#pragma unroll
              for (int i = 0; i < D; ++i)
                if (c[i] == m) c[i] += 1u, raised[i] += 1u;
              m += 1u;
            }
          } else {
            x -= 1;
            m = U32MAX;
#pragma unroll
            for (int i = 0; i < D; ++i) {
              const int64_t T = (int64_t)A[i] + (int64_t)x + (int64_t)O[i];
              if ((int64_t)c[i] > T) c[i] -= 1u;
              m = min(m, c[i]);
            }
          }
        }
        k.m = m;
        k.x = (uint32_t)x;
        k.e += k.rem;
        k.rem = 0;
        done = true;
      } else {
        done = replay_step<D, MODE>(a, k, e0, info, bits0, A, O, c, raised, ws, lut, rlut);
      }
      st_cyc += clock64() - t0;
      if (done) {
        const uint32_t L = info & 0x7fffffffu;
#pragma unroll
        for (int i = 0; i < D; ++i)
          if (MODE > 1 || !((bits0 >> i) & 1u))
            st_relaxed_u64(a.slim64 + cells[i], ((unsigned long long)(rank[i] + L) << 32) | c[i]);
        has = false;
        ++st_runs;
        if (a.trace) a.trace[3ull * rid + 2] = gtimer();
      }
      progressed = true;
    }
    if (__any_sync(0xffffffffu, progressed)) {
      idle = 0;
    } else if (++idle > SFK_IDLE_SPINS) {
      if (SFK_IDLE_MAX_NS) __nanosleep(min(idle * 4u, (uint32_t)SFK_IDLE_MAX_NS));
    }
  }
#pragma unroll
  for (int i = 0; i < D; ++i) {
    unsigned long long r = raised[i];
    for (int off = 16; off > 0; off >>= 1) r += __shfl_down_sync(0xffffffffu, r, off);
    if (lane == 0 && r) atomicAdd(a.inc + i, r);
  }
  // diagnostics (sfk_engine_stats): words by replay path, replay cycles, runs, warp iterations
  unsigned long long sv[8] = {ws[0], ws[1], ws[2], (unsigned long long)st_cyc, st_runs, lane == 0 ? st_iters : 0ull,
                              ws[3], ws[4]};
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    unsigned long long v = sv[q];
    for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
    if (lane == 0 && v) atomicAdd(&g_engine_stats[q], v);
  }
}

__global__ void pack_slim_k(const uint32_t* __restrict__ slim, unsigned long long* __restrict__ s64, uint32_t cells) {
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < cells; c += gridDim.x * blockDim.x) s64[c] = slim[c];
}
__global__ void unpack_slim_k(const unsigned long long* __restrict__ s64, uint32_t* __restrict__ slim, uint32_t cells) {
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < cells; c += gridDim.x * blockDim.x)
    slim[c] = (uint32_t)s64[c];
}

__global__ void ctl_init_k(Ctl* ctl) {
  ctl->fail_t = NONE32;
  ctl->n_runs = 0;
  ctl->n_ins = 0;
  ctl->qhead = 0;
  ctl->qtail = 0;
  ctl->executed = 0;
  ctl->bad_op = NONE32;
}

// undo the fat deltas of ops t >= t* (the fat was written for the whole
// batch; u32 arithmetic is modular so the correction is exact)
template <int D, int KIND>
__global__ void fat_undo_k(HashArgs<D> a, uint32_t* __restrict__ fat, uint32_t zstride) {
  const uint32_t tstar = a.ctl->fail_t;
  if (tstar == NONE32) return;
  for (int64_t t = (int64_t)tstar + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < a.n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = load_key(a.keys, t);
    const uint32_t undo = a.ops[t] ? 1u : 0xFFFFFFFFu;
#pragma unroll
    for (int i = 0; i < D; ++i) {
      uint32_t cell = (uint32_t)i * a.row_cells + (uint32_t)bucket(key, a.cell_seeds.s[i], a.cm);
      uint32_t k = (KIND == 0) ? (uint32_t)bucket(key, a.slot_seeds.s[i], a.zm) : 0u;
      atomicAdd(fat + (size_t)cell * zstride + k, undo);
    }
  }
}

// result = {status, op_index, n_ins}; CM tallies (+n_ins per row)
__global__ void finalize_k(const Ctl* ctl, const uint8_t* __restrict__ ops, int variant_kind, int64_t* result,
                           unsigned long long* inc, int d, int cm_tallies) {
  if (ctl->bad_op != NONE32) {
    result[0] = SFK_BAD_OPCODE;
    result[1] = (int64_t)ctl->bad_op;
    result[2] = 0;
    return;
  }
  const uint32_t ts = ctl->fail_t;
  int64_t status = SFK_OK;
  if (ts != NONE32) {
    const int op = ops[ts];
    // variant_kind: 0 SF1 / CU (delete unsupported), 1 SFF / CM (delete phantom)
    status = op == 0 ? SFK_SATURATED : (variant_kind == 0 ? SFK_UNSUPPORTED : SFK_PHANTOM);
  }
  result[0] = status;
  result[1] = ts == NONE32 ? -1 : (int64_t)ts;
  result[2] = (int64_t)ctl->n_ins;
  if (cm_tallies)
    for (int i = 0; i < d; ++i) inc[i] += ctl->n_ins;
}

// inserts applied before the first failing op (CM exact path)
__global__ void count_ins_k(const uint8_t* __restrict__ ops, int64_t n, Ctl* ctl) {
  const uint32_t ts = ctl->fail_t;
  const int64_t lim = ts == NONE32 ? n : (int64_t)ts;
  unsigned long long ins = 0;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < lim; t += (int64_t)gridDim.x * blockDim.x)
    ins += ops[t] == 0;
  for (int off = 16; off > 0; off >>= 1) ins += __shfl_down_sync(0xffffffffu, ins, off);
  if ((threadIdx.x & 31) == 0 && ins) atomicAdd(&ctl->n_ins, ins);
}

// ---------------------------------------------------------------- CM fast path
// warp-aggregated atomics: lanes hitting the same cell merge their net delta
// (__match_any_sync) and the group leader issues one atomicAdd.
template <int D>
__global__ void __launch_bounds__(256) cm_atomic_k(uint32_t* __restrict__ counters, Seeds<D> seeds, Mod wm, uint32_t w,
                                                   const uint8_t* __restrict__ ops, KeySrc keys, int64_t n,
                                                   const Ctl* ctl) {
  // Two aggregation levels before a global atomic:
  //   * warp: the lanes of a 32-op group with the same cell merge (match_any);
  //   * block: a direct-mapped shared-memory table claims a slot for the
  //     first cell that hashes to it and sums every later update of that
  //     cell in shared memory; a cell whose slot is taken goes to L2 as
  //     before. A Zipf-hot cell appears within the first ops a block sees,
  //     so its updates (otherwise serialised on one L2 address) become one
  //     atomic per block at the end.
  // CM sums commute and the host precheck rules out saturation and
  // phantoms, so the order of the updates does not matter.
  constexpr int CM_UNR = 4;
  constexpr int CM_SLOTS = 4096;
  constexpr uint32_t EMPTY = 0xFFFFFFFFu;
  __shared__ uint32_t tag[CM_SLOTS];
  __shared__ int32_t cnt[CM_SLOTS];
  for (int q = threadIdx.x; q < CM_SLOTS; q += blockDim.x) tag[q] = EMPTY, cnt[q] = 0;
  __syncthreads();
  const int64_t limit = ctl ? (ctl->fail_t == NONE32 ? n : (int64_t)ctl->fail_t) : n;
  const int lane = threadIdx.x & 31;
  const int64_t warp_id = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = warp_id * 32 * CM_UNR; base < limit; base += nwarps * 32 * CM_UNR) {
    uint64_t key[CM_UNR];
    uint32_t op[CM_UNR];
#pragma unroll
    for (int u = 0; u < CM_UNR; ++u) {
      const int64_t t = base + u * 32 + lane;
      key[u] = t < limit ? load_key(keys, t) : 0ull;
      op[u] = t < limit ? ops[t] : 0u;
    }
#pragma unroll
    for (int u = 0; u < CM_UNR; ++u) {
      const int64_t t = base + u * 32 + lane;
      const bool active = t < limit;
      const unsigned amask = __ballot_sync(0xffffffffu, active);
      if (!active) continue;
      const unsigned del = __ballot_sync(amask, op[u] != 0);
#pragma unroll
      for (int i = 0; i < D; ++i) {
        const uint32_t cell = (uint32_t)i * w + (uint32_t)bucket(key[u], seeds.s[i], wm);
        const unsigned g = __match_any_sync(amask, cell);
        if (lane == __ffs(g) - 1) {
          const int net = __popc(g & ~del) - __popc(g & del);
          if (net) {
            const uint32_t slot = (cell * 0x9E3779B1u) >> (32 - 12);  // log2(CM_SLOTS) = 12
            uint32_t tg = tag[slot];
            if (tg == EMPTY) {
              const uint32_t old = atomicCAS(&tag[slot], EMPTY, cell);
              tg = old == EMPTY ? cell : old;
            }
            if (tg == cell) atomicAdd(&cnt[slot], net);
            else atomicAdd(counters + cell, (uint32_t)net);
          }
        }
      }
    }
  }
  __syncthreads();
  for (int q = threadIdx.x; q < CM_SLOTS; q += blockDim.x) {
    const uint32_t tg = tag[q];
    const int32_t c = cnt[q];
    if (tg != EMPTY && c) atomicAdd(counters + tg, (uint32_t)c);
  }
}


__global__ void stats_ops_k(const uint8_t* __restrict__ ops, int64_t n, Stats* st) {
  unsigned long long ins = 0, del = 0, fd = 0xFFFFFFFFFFFFFFFFull, fb = 0xFFFFFFFFFFFFFFFFull;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const uint8_t o = ops[t];
    if (o) { ++del; if ((unsigned long long)t < fd) fd = t; }
    else ++ins;
    if (o > 1 && (unsigned long long)t < fb) fb = t;
  }
  for (int off = 16; off > 0; off >>= 1) {
    ins += __shfl_down_sync(0xffffffffu, ins, off);
    del += __shfl_down_sync(0xffffffffu, del, off);
    fd = min(fd, __shfl_down_sync(0xffffffffu, fd, off));
    fb = min(fb, __shfl_down_sync(0xffffffffu, fb, off));
  }
  if ((threadIdx.x & 31) == 0) {
    if (ins) atomicAdd(&st->n_ins, ins);
    if (del) atomicAdd(&st->n_del, del);
    if (fd != 0xFFFFFFFFFFFFFFFFull) atomicMin(&st->first_del, fd);
    if (fb != 0xFFFFFFFFFFFFFFFFull) atomicMin(&st->first_bad, fb);
  }
}
__global__ void stats_ins_before_k(const uint8_t* __restrict__ ops, Stats* st) {
  const unsigned long long lim = st->first_del;
  unsigned long long ins = 0;
  for (unsigned long long t = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; t < lim;
       t += (unsigned long long)gridDim.x * blockDim.x)
    ins += ops[t] == 0;
  for (int off = 16; off > 0; off >>= 1) ins += __shfl_down_sync(0xffffffffu, ins, off);
  if ((threadIdx.x & 31) == 0 && ins) atomicAdd(&st->ins_before_first_del, ins);
}
// bias = 0x80000000 maps int32 counters onto u32 order (Count sketch)
__global__ void stats_counters_k(const uint32_t* __restrict__ c, int64_t cells, Stats* st, uint32_t bias) {
  uint32_t mx = 0, mn = U32MAX;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < cells; k += (int64_t)gridDim.x * blockDim.x) {
    mx = max(mx, c[k] ^ bias);
    mn = min(mn, c[k] ^ bias);
  }
  for (int off = 16; off > 0; off >>= 1) {
    mx = max(mx, __shfl_down_sync(0xffffffffu, mx, off));
    mn = min(mn, __shfl_down_sync(0xffffffffu, mn, off));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&st->cmax, mx);
    atomicMin(&st->cmin, mn);
  }
}

// ================================================================ host side
constexpr uint32_t SORT_FORK_MAX_ROWS = 8;  // sort_pairs: rows sorted concurrently

struct Plan {
  // sizes
  uint32_t n, N;  // ops, pairs (D*n)
  int D, kb;
  size_t cub_sort_bytes, cub_scan_bytes;
  uint32_t ntiles;
};

static size_t sort_temp_bytes(uint32_t N) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)N, 0, 32);
  return bytes;
}
static size_t scan_temp_bytes(uint32_t n) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)n);
  return bytes;
}

static size_t key_sort_temp_bytes(uint32_t n) {
  size_t a = 0, b = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, a, (const uint64_t*)nullptr, (uint64_t*)nullptr, (const uint32_t*)nullptr,
                                  (uint32_t*)nullptr, (int)n, 0, 64);
  cub::DeviceScan::InclusiveScan(nullptr, b, (const uint32_t*)nullptr, (uint32_t*)nullptr, cub::Max(), (int)n);
  return std::max(a, b);
}

static int bits_for(uint64_t v) {  // bits needed to represent values < v
  int b = 0;
  while (b < 64 && (1ull << b) < v) ++b;
  return b;
}

// Workspace layout shared by every parallel apply. Sizes are upper bounds
// for the given (kind, dims, n); a null base only measures.
struct Layout {
  uint32_t *k_in, *v_in, *k_out, *v_out;
  void* cub_tmp;
  size_t cub_tmp_bytes;
  void* tiles;        // SegState<Z> per tile
  uint32_t* fat_snap;
  uint32_t* fat_perm;  // SF3: the fat regrouped into fold-group order
  uint32_t* obs;
  uint2* obs2;
  uint32_t* delbits;
  uint32_t* wsum;
  uint32_t* wowner;
  WalkPiece* piece[3];
  RowMap* rmap[3];
  uint2* links;
  uint8_t* opflags;
  uint32_t* opdata;
  uint32_t* headflag;
  uint32_t *bnd, *bidx, *bpos, *isdel, *delpre;
  uint32_t* ridx;
  uint64_t *k64a, *k64b;          // SF1 ignore pass: materialised keys, sorted
  unsigned long long* htab;       //   key -> group id table (64-bit keys)
  uint32_t *ta, *tb, *headpos;     //   op ids, sorted op ids, key segment heads
  uint2* meta;                     //   per op: {key count, previous op of the same key}
  uint32_t* dmask;                 //   per op: a byte of dropped rows (D <= 8)
  uint32_t *rbrk, *hbits;          //   per op bits: a kept pair breaks the key's run / run head
  uint32_t* hbitsj;                //   run heads as bits by key-order position
  uint32_t* owner;                 // SF1 shared-cell fat phase: first claimant per fat cell
  uint8_t* shared;                 //   fat cells claimed by two or more keys
  uint32_t *ncnt, *noff;           //   per op: rows on shared cells, their exclusive prefix sums
  uint8_t* ign;                    //   dropped (op, row) flags in cell order
  void* ftiles;                    //   filtered-link scan tile carries
  void* recs;
  unsigned long long* slim64;
  uint8_t* zops;                   // oracle-assisted: an all-insert op stream
  uint32_t *omax0, *omax1;         // gated kinds: largest cap per 32 / 1024 ops
  uint32_t *brk, *brkpre;          // oracle-assisted: cap-break flags and their prefix counts
  int64_t* inc_scratch;            // CML: the engine's per-row raise tallies (discarded)
  Ctl* ctl;
  Stats* stats;
  size_t total;
  bool ok;
};

// kind: 0 SFF (bucketed), 1 SF1 (flat), 2 CU, 3 CM exact, 4 SF4 (bucketed, sum
// trigger), 5 SF3 (fold groups as buckets), 6 SF2 (flat fat + deletion sub-sketch),
// 7 CML (u16 exponents widened into fat_snap), 8 oracle-assisted slim
// (7 and 8: insert-only gated min-raise with a per-op gate, op-by-op replay)
static uint64_t runrec_bytes(int d) {
  switch (d) {
    case 1: return sizeof(RunRec<1>);
    case 2: return sizeof(RunRec<2>);
    case 3: return sizeof(RunRec<3>);
    case 4: return sizeof(RunRec<4>);
    case 5: return sizeof(RunRec<5>);
    case 6: return sizeof(RunRec<6>);
    case 7: return sizeof(RunRec<7>);
    default: return sizeof(RunRec<8>);
  }
}

// bytes of run_scan's tile buffer for N pairs (any z <= 8)
static size_t scan_tiles_bytes(uint64_t N) {
  const uint64_t ntiles = (N + SCAN_TILE - 1) / SCAN_TILE;
  size_t tbytes = 0;
  cub::DeviceScan::ExclusiveScan(nullptr, tbytes, (SegState<8>*)nullptr, (SegState<8>*)nullptr, SegStateOp<8>(),
                                 seg_identity<8>(), (int)std::max<uint64_t>(ntiles, 1));
  return 2 * ntiles * sizeof(SegState<8>) + 256 + tbytes + 256;
}

// bytes of the filtered-link scan's tile buffer for N pairs
static size_t filt_tiles_bytes(uint64_t N) {
  const uint64_t ntiles = (N + SCAN_TILE - 1) / SCAN_TILE;
  size_t tbytes = 0;
  cub::DeviceScan::ExclusiveScan(nullptr, tbytes, (SegCnt*)nullptr, (SegCnt*)nullptr, SegCntOp(),
                                 SegCnt{0u, 0u, NONE32}, (int)std::max<uint64_t>(ntiles, 1));
  return 2 * ntiles * sizeof(SegCnt) + 256 + tbytes + 256;
}

static Layout carve(void* base, size_t cap, int kind, int d, int64_t w, int64_t wp, int z, int64_t n) {
  Carver cv(base, cap);
  Layout L{};
  const uint64_t N = (uint64_t)d * (uint64_t)n;
  L.ctl = cv.take<Ctl>(1);
  L.stats = cv.take<Stats>(1);
  L.k_in = cv.take<uint32_t>(N);
  L.v_in = cv.take<uint32_t>(N);
  L.k_out = cv.take<uint32_t>(N);
  L.v_out = cv.take<uint32_t>(N);
  L.cub_tmp_bytes = std::max(sort_temp_bytes((uint32_t)N), scan_temp_bytes((uint32_t)n + 1));
  if (kind == 1 || kind == 2) L.cub_tmp_bytes = std::max(L.cub_tmp_bytes, key_sort_temp_bytes((uint32_t)n));
  // room for the d concurrent per-row sorts of sort_pairs (a few KB over one sort of all pairs)
  if (d > 1 && d <= (int)SORT_FORK_MAX_ROWS)
    L.cub_tmp_bytes = std::max(L.cub_tmp_bytes, (size_t)d * ((sort_temp_bytes((uint32_t)n) + 255) & ~(size_t)255));
  L.cub_tmp = cv.take<char>(L.cub_tmp_bytes);
  const uint64_t ntiles = (N + SCAN_TILE - 1) / SCAN_TILE;
  L.tiles = cv.take<char>(scan_tiles_bytes(N));
  const bool bucketed = kind == 0 || kind == 4 || kind == 5;
  const bool gated = kind == 7 || kind == 8;
  const bool deletes = bucketed || kind == 6 || gated;  // runs carry delete bits (and observations)
  uint64_t fat_cells = 0;
  if (bucketed) fat_cells = (uint64_t)d * w * z;
  if (kind == 1 || kind == 6) fat_cells = std::max((uint64_t)d * wp, (uint64_t)d * w);
  if (kind == 3 || kind == 7) fat_cells = (uint64_t)d * w;
  L.fat_snap = cv.take<uint32_t>(fat_cells ? fat_cells : 1);
  L.fat_perm = cv.take<uint32_t>(kind == 5 ? fat_cells : 1);
  const bool need_obs = kind == 1 || kind == 2 || kind == 6 || gated;
  L.obs = cv.take<uint32_t>(need_obs ? (uint64_t)n : 1);  // per-op b_min
  L.obs2 = cv.take<uint2>(1);  // SFF interleaves its observations with the links
  L.delbits = cv.take<uint32_t>(deletes ? n / 32 + 16 : 1);
  L.wsum = cv.take<uint32_t>(kind == 0 ? n / 32 + 32 : 1);
  {
    const uint64_t nw = (kind == 0 || kind == 4 || kind == 5) ? n / 32 + 32 : 1;  // long-run maps
    L.wowner = cv.take<uint32_t>(nw);
    for (int lv = 0; lv < MAP_LEVELS; ++lv) {
      const uint64_t cnt = nw > 1 ? (nw >> (5 * lv)) + 1 : 1;
      L.piece[lv] = cv.take<WalkPiece>(cnt);
      L.rmap[lv] = cv.take<RowMap>(cnt * (uint64_t)d);
    }
  }
  const bool engine = kind != 3;
  L.links = cv.take<uint2>(engine ? 4 * N : 1);
  L.opflags = cv.take<uint8_t>(engine ? n : 1);
  L.opdata = cv.take<uint32_t>(need_obs ? (uint64_t)n : 1);
  L.headflag = cv.take<uint32_t>(engine ? n : 1);
  L.bnd = cv.take<uint32_t>(engine ? n + 1 : 1);
  L.bidx = cv.take<uint32_t>(engine ? n + 1 : 1);
  L.bpos = cv.take<uint32_t>(engine ? n + 2 : 1);
  L.isdel = cv.take<uint32_t>(engine ? n + 1 : 1);
  L.delpre = cv.take<uint32_t>(engine ? n + 1 : 1);
  L.ridx = cv.take<uint32_t>(engine ? n : 1);
  {
    const bool sf1 = kind == 1 || kind == 2;  // SF1 and CU: the ignore pass
    L.meta = cv.take<uint2>(sf1 ? n : 1);
    L.dmask = cv.take<uint32_t>(sf1 ? (uint64_t)n / 4 + 1 : 1);
    L.rbrk = cv.take<uint32_t>(sf1 ? (uint64_t)n / 32 + 1 : 1);
    L.hbits = cv.take<uint32_t>(sf1 ? (uint64_t)n / 32 + 1 : 1);
    L.hbitsj = cv.take<uint32_t>(sf1 ? (uint64_t)n / 32 + 1 : 1);
    const bool f1 = kind == 1;
    L.owner = cv.take<uint32_t>(f1 ? (uint64_t)d * wp : 1);
    L.shared = cv.take<uint8_t>(f1 ? (uint64_t)d * wp : 1);
    L.ncnt = cv.take<uint32_t>(f1 ? (uint64_t)n + 1 : 1);
    L.noff = cv.take<uint32_t>(f1 ? (uint64_t)n + 1 : 1);
    L.k64a = cv.take<uint64_t>(sf1 ? n : 1);
    L.k64b = cv.take<uint64_t>(sf1 ? n : 1);
    L.htab = cv.take<unsigned long long>(sf1 ? slot_cap((uint32_t)std::max<int64_t>(n, 1)) : 1);
    L.ta = cv.take<uint32_t>(sf1 ? n : 1);
    L.tb = cv.take<uint32_t>(sf1 ? n : 1);
    L.headpos = cv.take<uint32_t>(sf1 ? n : 1);
    L.ign = cv.take<uint8_t>(sf1 ? N : 1);
    L.ftiles = cv.take<char>(sf1 ? filt_tiles_bytes(N) : 1);
  }
  L.recs = cv.take<char>(engine ? (uint64_t)n * runrec_bytes(d) : 1);
  L.slim64 = cv.take<unsigned long long>(engine ? (uint64_t)d * w : 1);
  L.zops = cv.take<uint8_t>(kind == 8 ? (uint64_t)n : 1);
  L.omax0 = cv.take<uint32_t>(gated ? n / 32 + 2 : 1);
  L.omax1 = cv.take<uint32_t>(gated ? n / 1024 + 2 : 1);
  L.brk = cv.take<uint32_t>(kind == 8 ? n + 1 : 1);
  L.brkpre = cv.take<uint32_t>(kind == 8 ? n + 1 : 1);
  L.inc_scratch = cv.take<int64_t>(MAXSEEDS);
  L.total = cv.off + 256;
  L.ok = cv.ok;
  return L;
}

// optional per-run engine trace (diagnostics; SFK_ENGINE_TRACE=1)
static unsigned long long* g_trace = nullptr;
static uint32_t g_trace_cap = 0;

int engine_trace(unsigned long long* host_out, size_t runs) {
  if (!g_trace) return -1;
  const size_t m = runs < g_trace_cap ? runs : g_trace_cap;
  return (int)cudaMemcpy(host_out, g_trace, sizeof(unsigned long long) * 3 * m, cudaMemcpyDeviceToHost);
}

// optional CUDA-event timing of the engine kernel (bench instrumentation)
static bool g_time_engine = false;
static bool g_ev_pending = false;
static cudaEvent_t g_ev[2];

int engine_timing(int on) {
  if (on && !g_time_engine) {
    cudaEventCreate(&g_ev[0]);
    cudaEventCreate(&g_ev[1]);
  }
  g_time_engine = on != 0;
  g_ev_pending = false;
  return 0;
}

// elapsed ms of the last timed engine launch (synchronises on it); -1 if none
float engine_last_ms() {
  if (!g_ev_pending) return -1.0f;
  float ms = -1.0f;
  if (cudaEventSynchronize(g_ev[1]) == cudaSuccess) cudaEventElapsedTime(&ms, g_ev[0], g_ev[1]);
  g_ev_pending = false;
  return ms;
}

int engine_stats(unsigned long long* out, int reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out, g_engine_stats, sizeof(unsigned long long) * 8);
  if (e == cudaSuccess && reset) {
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    e = cudaMemcpyToSymbol(g_engine_stats, z, sizeof(z));
  }
  return (int)e;
}

size_t parallel_workspace_size(int kind, int d, int64_t w, int64_t wp, int z, int64_t n) {
  if (n <= 0) return 256;
  Layout L = carve(nullptr, ~size_t(0), kind, d, w, wp, z, n);
  return L.total;
}

template <int Z, bool HAS_FAT, int OBS, bool LINKS>
static int run_scan(const uint32_t* keys, const uint32_t* vals, uint32_t N, int kb, void* tiles, ScanOut so,
                    cudaStream_t st) {
  const uint32_t ntiles = (N + SCAN_TILE - 1) / SCAN_TILE;
  // tiles: [tile aggregates][their exclusive prefixes][the scan's temp storage]
  SegState<Z>* ta = static_cast<SegState<Z>*>(tiles);
  SegState<Z>* tb = ta + ntiles;
  void* tmp = reinterpret_cast<void*>((reinterpret_cast<uintptr_t>(tb + ntiles) + 255) & ~uintptr_t(255));
  { note_launch(); segscan_reduce_k<Z, HAS_FAT><<<ntiles, SCAN_THREADS, 0, st>>>(keys, vals, N, kb, ta); }
  // the tile carries: a multi-block decoupled look-back scan (one CTA scanning
  // 23K 24-B states in a loop took ~0.12 ms per cfg-3 build)
  size_t tbytes = 0;
  cub::DeviceScan::ExclusiveScan(nullptr, tbytes, ta, tb, SegStateOp<Z>(), seg_identity<Z>(), (int)ntiles, st);
  cudaError_t e = cub::DeviceScan::ExclusiveScan(tmp, tbytes, ta, tb, SegStateOp<Z>(), seg_identity<Z>(), (int)ntiles, st);
  if (e != cudaSuccess) {
    set_error("segscan tiles: %s", cudaGetErrorString(e));
    return (int)e;
  }
  { note_launch(); segscan_apply_k<Z, HAS_FAT, OBS, LINKS><<<ntiles, SCAN_THREADS, 0, st>>>(keys, vals, N, kb, tb, so); }
  return check_launch("segscan");
}


template <bool HAS_FAT, int OBS, bool LINKS>
static int run_scan_z(int z, const uint32_t* keys, const uint32_t* vals, uint32_t N, int kb, void* tiles, ScanOut so,
                      cudaStream_t st) {
  switch (z) {
    case 1: return run_scan<1, HAS_FAT, OBS, LINKS>(keys, vals, N, kb, tiles, so, st);
    case 2: return run_scan<2, HAS_FAT, OBS, LINKS>(keys, vals, N, kb, tiles, so, st);
    case 3: return run_scan<3, HAS_FAT, OBS, LINKS>(keys, vals, N, kb, tiles, so, st);
    case 4: return run_scan<4, HAS_FAT, OBS, LINKS>(keys, vals, N, kb, tiles, so, st);
    case 5: return run_scan<5, HAS_FAT, OBS, LINKS>(keys, vals, N, kb, tiles, so, st);
    case 6: return run_scan<6, HAS_FAT, OBS, LINKS>(keys, vals, N, kb, tiles, so, st);
    case 7: return run_scan<7, HAS_FAT, OBS, LINKS>(keys, vals, N, kb, tiles, so, st);
    case 8: return run_scan<8, HAS_FAT, OBS, LINKS>(keys, vals, N, kb, tiles, so, st);
  }
  set_error("segscan: unsupported z=%d", z);
  return 1;
}

// Stable sort of the (cell, t|op|slot) pairs by cell. The pairs of row i sit
// at [i n, (i + 1) n) and every cell of row i lies in [i R, (i + 1) R) (R
// cells per row), so when R is a power of two each row sorts on its own over
// log2(R) bits: for cfg 3 two 8-bit onesweep passes instead of three for the
// 18-bit cells of all rows together.
//
// A row's sort alone leaves most of HBM idle (onesweep over 12M pairs: ~1.7
// TB/s per pass, its tiles chained by the decoupled look-back), so large rows
// sort concurrently, one side stream and one slice of the CUB workspace per
// row, forked from and joined back into `st` with events. The side streams
// and events are per host thread and device, so concurrent callers never
// share an event.
constexpr uint32_t SORT_FORK_MIN_PAIRS = 1u << 20;  // per row
struct SortFork {
  cudaStream_t s[SORT_FORK_MAX_ROWS] = {};
  cudaEvent_t ev[SORT_FORK_MAX_ROWS + 1] = {};
  bool ok = false, tried = false;
};
static SortFork* sort_fork() {
  thread_local SortFork forks[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  SortFork& f = forks[dev];
  if (!f.tried) {
    f.tried = true;
    f.ok = true;
    for (uint32_t i = 0; i < SORT_FORK_MAX_ROWS && f.ok; ++i)
      f.ok = cudaStreamCreateWithFlags(&f.s[i], cudaStreamNonBlocking) == cudaSuccess;
    for (uint32_t i = 0; i <= SORT_FORK_MAX_ROWS && f.ok; ++i)
      f.ok = cudaEventCreateWithFlags(&f.ev[i], cudaEventDisableTiming) == cudaSuccess;
    if (!f.ok) cudaGetLastError();
  }
  return f.ok ? &f : nullptr;
}
static bool sort_fork_enabled() {
  static const int v = [] {
    const char* s = getenv("SFK_SORT_FORK");
    return s ? atoi(s) : 1;
  }();
  return v != 0;
}

static int sort_pairs(Layout& L, uint32_t N, uint32_t rows, uint64_t row_cells, cudaStream_t st) {
  size_t bytes = L.cub_tmp_bytes;
  cudaError_t e = cudaSuccess;
  const int row_bits = bits_for(row_cells);
  const int all_bits = bits_for((uint64_t)rows * row_cells);
  const bool per_row = rows > 1 && (row_cells & (row_cells - 1)) == 0 && (row_bits + 7) / 8 < (all_bits + 7) / 8;
  if (per_row) {
    const uint32_t n = N / rows;
    size_t row_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, row_bytes, L.k_in, L.k_out, L.v_in, L.v_out, (int)n, 0,
                                    std::max(row_bits, 1), st);
    row_bytes = (row_bytes + 255) & ~(size_t)255;
    SortFork* f = (sort_fork_enabled() && rows <= SORT_FORK_MAX_ROWS && n >= SORT_FORK_MIN_PAIRS &&
                   row_bytes * rows <= L.cub_tmp_bytes)
                      ? sort_fork()
                      : nullptr;
    if (f) {
      e = cudaEventRecord(f->ev[SORT_FORK_MAX_ROWS], st);
      for (uint32_t i = 0; i < rows && e == cudaSuccess; ++i) {
        const size_t o = (size_t)i * n;
        size_t b = row_bytes;
        e = cudaStreamWaitEvent(f->s[i], f->ev[SORT_FORK_MAX_ROWS], 0);
        if (e == cudaSuccess)
          e = cub::DeviceRadixSort::SortPairs(static_cast<char*>(L.cub_tmp) + i * row_bytes, b, L.k_in + o,
                                              L.k_out + o, L.v_in + o, L.v_out + o, (int)n, 0,
                                              std::max(row_bits, 1), f->s[i]);
        if (e == cudaSuccess) e = cudaEventRecord(f->ev[i], f->s[i]);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(st, f->ev[i], 0);
      }
      if (e != cudaSuccess) {
        set_error("radix sort (forked rows): %s", cudaGetErrorString(e));
        return (int)e;
      }
      return 0;
    }
    for (uint32_t i = 0; i < rows && e == cudaSuccess; ++i) {
      const size_t o = (size_t)i * n;
      e = cub::DeviceRadixSort::SortPairs(L.cub_tmp, bytes, L.k_in + o, L.k_out + o, L.v_in + o, L.v_out + o, (int)n, 0,
                                          std::max(row_bits, 1), st);
    }
  } else {
    e = cub::DeviceRadixSort::SortPairs(L.cub_tmp, bytes, L.k_in, L.k_out, L.v_in, L.v_out, (int)N, 0,
                                        std::max(all_bits, 1), st);
  }
  if (e != cudaSuccess) {
    set_error("radix sort: %s", cudaGetErrorString(e));
    return (int)e;
  }
  return 0;
}

template <int D>
static HashArgs<D> make_hash(KeySrc ks, const uint8_t* ops, int64_t n, const uint64_t* cell_seeds,
                             const uint64_t* slot_seeds, uint64_t row_cells, int z, int kb, Layout& L,
                             int unsupported_deletes) {
  HashArgs<D> h;
  h.keys = ks;
  h.ops = ops;
  h.n = n;
  for (int i = 0; i < D; ++i) {
    h.cell_seeds.s[i] = cell_seeds[i];
    h.slot_seeds.s[i] = slot_seeds ? slot_seeds[i] : 0;
  }
  h.cm = make_mod(row_cells);
  h.zm = make_mod((uint64_t)std::max(z, 1));
  h.row_cells = (uint32_t)row_cells;
  h.kb = kb;
  h.key_out = L.k_in;
  h.val_out = L.v_in;
  h.unsupported_deletes = unsupported_deletes;
  h.pos = nullptr;
  h.ctl = L.ctl;
  return h;
}

// brk[e] = 1 when op e's cap does not exceed op e-1's (row-0 order); brk[n] = 0
__global__ void cap_break_k(const uint32_t* __restrict__ opdata, uint32_t n, uint32_t* __restrict__ brk) {
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e <= n; e += gridDim.x * blockDim.x)
    brk[e] = (e == 0 || e == n) ? (e == 0 ? 1u : 0u) : (opdata[e] <= opdata[e - 1] ? 1u : 0u);
}
// per 32-op word (row-0 order) the largest cap, then per 1024 ops
__global__ void opmax_word_k(const uint32_t* __restrict__ opdata, uint32_t n, uint32_t* __restrict__ omax0) {
  const uint32_t lane = threadIdx.x & 31u;
  for (uint32_t e0 = (blockIdx.x * blockDim.x + threadIdx.x) & ~31u; e0 < n; e0 += gridDim.x * blockDim.x) {
    const uint32_t e = e0 + lane;
    uint32_t v = e < n ? opdata[e] : 0u;
    for (int off = 16; off > 0; off >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, off));
    if (lane == 0) omax0[e0 >> 5] = v;
  }
}
__global__ void opmax_block_k(const uint32_t* __restrict__ omax0, uint32_t nwords, uint32_t* __restrict__ omax1) {
  const uint32_t lane = threadIdx.x & 31u;
  for (uint32_t w0 = (blockIdx.x * blockDim.x + threadIdx.x) & ~31u; w0 < nwords; w0 += gridDim.x * blockDim.x) {
    const uint32_t w = w0 + lane;
    uint32_t v = w < nwords ? omax0[w] : 0u;
    for (int off = 16; off > 0; off >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, off));
    if (lane == 0) omax1[w0 >> 5] = v;
  }
}

// The run/engine tail shared by SFF, SF1 and CU once the row-0 sorted slim
// pairs (k_out/v_out), the links and the observations exist.
template <int D, int MODE>
static int run_engine(Layout& L, uint32_t* slim, const uint64_t* slim_seeds, int64_t w, KeySrc ks, uint32_t n, int kb,
                      int64_t* inc, cudaStream_t st, bool b_opdata = false, bool has_ign = false,
                      bool cap_skip = false, bool cap_mono = false) {
  const int sms = sm_count();
  RunArgs<D> ra;
  ra.vals0 = L.v_out;
  ra.kb = kb;
  ra.n = n;
  ra.links = L.links;
  ra.lstride = 4;
  ra.obs = (MODE == 0 || b_opdata) ? L.obs : nullptr;
  ra.keys = ks;
  ra.opflags = L.opflags;
  ra.opdata = L.opdata;
  ra.headflag = L.headflag;
  ra.delbits = MODE >= 2 ? L.delbits : nullptr;
  ra.bnd = L.bnd;
  ra.isdel = L.isdel;
  ra.order = has_ign ? L.tb : nullptr;
  ra.obs_by_pos = 0;
  ra.cbk = (MODE == 0 && has_ign) ? reinterpret_cast<const uint4*>(L.k64a) : nullptr;  // (sf1_ignore_pass's cb)
  ra.hbits = has_ign ? L.hbits : nullptr;
  ra.ctl = L.ctl;
  // (with dropped pairs the ignore pass has decided the run heads: runs_head_ign_k)
  if (!has_ign) { note_launch(); runs_head_k<D><<<grid_for(n, 256, sms * 16), 256, 0, st>>>(ra); }
  { note_launch(); runs_mark_k<D><<<grid_for(n, 256, sms * 16), 256, 0, st>>>(ra); }
  size_t bytes = L.cub_tmp_bytes;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(L.cub_tmp, bytes, L.headflag, L.ridx, (int)n, st);
  // run extents: boundaries (row-0 order) and delete prefix counts
  cudaMemsetAsync(L.isdel + n, 0, 4, st);
  if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(L.cub_tmp, bytes, L.bnd, L.bidx, (int)n, st);
  if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(L.cub_tmp, bytes, L.isdel, L.delpre, (int)n + 1, st);
  if (e != cudaSuccess) {
    set_error("run scan: %s", cudaGetErrorString(e));
    return (int)e;
  }
  { note_launch(); boundary_pos_k<<<grid_for(n, 256, sms * 16), 256, 0, st>>>(L.bnd, L.bidx, n, L.bpos); }
  BuildArgs<D> ba;
  ba.headflag = L.headflag;
  ba.ridx = L.ridx;
  ba.opflags = L.opflags;
  ba.bidx = L.bidx;
  ba.bpos = L.bpos;
  ba.delpre = L.delpre;
  ba.delbits = MODE >= 2 ? L.delbits : nullptr;
  ba.obs2 = MODE >= 2 ? L.links + 1 : nullptr;
  ba.links = L.links;
  ba.lstride = 4;
  ba.n = n;
  ba.keys = ks;
  for (int i = 0; i < D; ++i) ba.seeds.s[i] = slim_seeds[i];
  ba.wm = make_mod((uint64_t)w);
  ba.w = (uint32_t)w;
  ba.recs = static_cast<RunRec<D>*>(L.recs);
  ba.order = has_ign ? L.tb : nullptr;
  ba.dmask = has_ign ? reinterpret_cast<const uint8_t*>(L.dmask) : nullptr;
  ba.hbits = has_ign ? L.hbits : nullptr;
  ba.ctl = L.ctl;
  { note_launch(); runs_build_k<D><<<grid_for(n, 256, sms * 16), 256, 0, st>>>(ba); }
  const uint32_t cells = (uint32_t)(D * w);
  { note_launch(); pack_slim_k<<<grid_for(cells, 256, sms * 8), 256, 0, st>>>(slim, L.slim64, cells); }
  EngineArgs<D> ea;
  ea.slim64 = L.slim64;
  ea.recs = static_cast<const RunRec<D>*>(L.recs);
  ea.opdata = L.opdata;
  ea.delbits = L.delbits;
  ea.wsum = L.wsum;
  for (int lv = 0; lv < MAP_LEVELS; ++lv) ea.piece[lv] = nullptr, ea.rmap[lv] = nullptr;
  ea.omax[0] = ea.omax[1] = nullptr;
  if (cap_skip && !getenv("SFK_NO_CAP_SKIP")) {  // diagnostics knob: op-by-op only
    const uint32_t nwords = (n + 31) / 32;
    { note_launch(); opmax_word_k<<<grid_for(n, 256, sms * 8), 256, 0, st>>>(L.opdata, n, L.omax0); }
    { note_launch(); opmax_block_k<<<grid_for(nwords, 256, sms * 8), 256, 0, st>>>(L.omax0, nwords, L.omax1); }
    ea.omax[0] = L.omax0;
    ea.omax[1] = L.omax1;
  }
  ea.brk_pre = nullptr;
  if (cap_mono && !getenv("SFK_NO_CAP_SKIP")) {
    { note_launch(); cap_break_k<<<grid_for(n + 1, 256, sms * 8), 256, 0, st>>>(L.opdata, n, L.brk); }
    size_t bytes2 = L.cub_tmp_bytes;
    if (cub::DeviceScan::ExclusiveSum(L.cub_tmp, bytes2, L.brk, L.brkpre, (int)n + 1, st) != cudaSuccess) {
      set_error("cap break scan failed");
      return 1;
    }
    ea.brk_pre = L.brkpre;
  }
  if (MODE == 2 || (MODE == 3 && !b_opdata)) {
    const uint32_t nwords = (n + 31) / 32;
    const int sum_mode = MODE == 3 ? 1 : 0;
    if (MODE == 2) { note_launch(); word_sums_k<<<grid_for(nwords, 256, sms * 8), 256, 0, st>>>(L.delbits, nwords, L.wsum); }
    if (!getenv("SFK_NO_LONGRUN")) {  // diagnostics knob: the word-by-word replay only
      const RunRec<D>* rp = static_cast<const RunRec<D>*>(L.recs);
      { note_launch(); long_owner_k<D><<<sms * 8, 256, 0, st>>>(rp, L.ctl, L.wowner); }
      { note_launch(); word_maps_k<D><<<grid_for(nwords, 256, sms * 8), 256, 0, st>>>(rp, L.ctl, L.wowner, L.delbits, nwords, L.piece[0], L.rmap[0], sum_mode); }
      for (int lv = 1; lv < MAP_LEVELS; ++lv) {
        const uint32_t nb = nwords >> (5 * lv);
        if (nb) { note_launch(); block_maps_k<D><<<grid_for(nb, 256, sms * 8), 256, 0, st>>>(rp, L.ctl, L.wowner, nwords, 1u << (5 * lv), L.piece[lv - 1], L.rmap[lv - 1], L.piece[lv], L.rmap[lv], nb, sum_mode); }
      }
      for (int lv = 0; lv < MAP_LEVELS; ++lv) ea.piece[lv] = L.piece[lv], ea.rmap[lv] = L.rmap[lv];
    }
  }
  ea.ctl = L.ctl;
  ea.inc = reinterpret_cast<unsigned long long*>(inc);
  ea.budget = engine_budget();
  ea.b_opdata = b_opdata ? 1 : 0;
  ea.trace = nullptr;
  if (getenv("SFK_ENGINE_TRACE")) {  // diagnostics only: per-run timestamps
    if (g_trace_cap < n) {
      if (g_trace) cudaFree(g_trace);
      cudaMalloc(&g_trace, sizeof(unsigned long long) * 3 * (size_t)n);
      g_trace_cap = n;
    }
    ea.trace = g_trace;
  }
  if (g_time_engine) cudaEventRecord(g_ev[0], st);
  { note_launch(); poll_engine_k<D, MODE><<<sms * engine_blocks_per_sm(), SFK_ENGINE_THREADS, 0, st>>>(ea); }
  if (g_time_engine) {
    cudaEventRecord(g_ev[1], st);
    g_ev_pending = true;
  }
  { note_launch(); unpack_slim_k<<<grid_for(cells, 256, sms * 8), 256, 0, st>>>(L.slim64, slim, cells); }
  return check_launch("poll_engine");
}


// CML gate (_kernels.py:200-204): insert number pos = start_pos + t draws
// uf = (finalize64(rng_seed + (pos + 1) GOLDEN) >> 11) 2^-53 and raises when
// uf < base ** -c for the min exponent c. With gate[c] = base ** -c
// non-increasing (the caller checks), that is c < E_t where E_t = the first
// c with gate[c] <= uf: a per-op cap like SF1's b_min. Ops t >= t* are never
// replayed, and every op before t* is an insert, so pos = start_pos + t.
__global__ void cml_gate_k(const double* __restrict__ gate, uint64_t rng_seed, int64_t start_pos, uint32_t n,
                           uint32_t* __restrict__ obs) {
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const uint64_t pos = (uint64_t)(start_pos + (int64_t)t);
    const uint64_t u = mix64(rng_seed + (pos + 1ull) * 0x9E3779B97F4A7C15ull);
    const double uf = (double)(u >> 11) * (1.0 / 9007199254740992.0);
    uint32_t lo = 0, hi = 65536;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (__ldg(gate + mid) <= uf) hi = mid; else lo = mid + 1;
    }
    obs[t] = lo;
  }
}
// oracle-assisted cap (_kernels.py:400-405): raise when m < np.uint64(true
// count), so a negative count wraps to a cap above every u32 minimum; caps
// above 2^32 - 1 clamp to it (exact: the precheck keeps every cell below it)
__global__ void oracle_gate_k(const int64_t* __restrict__ tc, uint32_t n, uint32_t* __restrict__ obs) {
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const uint64_t v = (uint64_t)tc[t];
    obs[t] = v >= (uint64_t)U32MAX ? U32MAX : (uint32_t)v;
  }
}
__global__ void widen_u16_k(const uint16_t* __restrict__ src, uint32_t* __restrict__ dst, uint32_t cells) {
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < cells; c += gridDim.x * blockDim.x) dst[c] = src[c];
}
__global__ void narrow_u16_k(const uint32_t* __restrict__ src, uint16_t* __restrict__ dst, uint32_t cells) {
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < cells; c += gridDim.x * blockDim.x)
    dst[c] = (uint16_t)src[c];
}

// SF3 fat (d, w') with w' = z w: fold group of slim cell (i, j) = fat cells
// j + m w, m < z. Regrouped as (i, j, m) so the bucketed scan applies.
__global__ void fold_gather_k(const uint32_t* __restrict__ fat, uint32_t* __restrict__ grp, uint32_t d, uint32_t w,
                              uint32_t z) {
  const uint64_t total = (uint64_t)d * w * z;
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = q / ((uint64_t)w * z), r = q % ((uint64_t)w * z), j = r / z, m = r % z;
    grp[q] = fat[i * w * z + m * w + j];
  }
}
__global__ void fold_scatter_k(const uint32_t* __restrict__ grp, uint32_t* __restrict__ fat, uint32_t d, uint32_t w,
                               uint32_t z) {
  const uint64_t total = (uint64_t)d * w * z;
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = q / ((uint64_t)w * z), r = q % ((uint64_t)w * z), j = r / z, m = r % z;
    fat[i * w * z + m * w + j] = grp[q];
  }
}


// ---------------------------------------------------------------- SF1 fat phase over shared cells
// An SF1 op's post-op count on a fat cell that no other key of the batch
// touches is its fat value before the batch plus the key's count so far, so
// only the pairs on cells that two or more keys share (56 % at cfg 4) need
// the cell sort and the segmented scan. fat_owner_k lets every key's head
// claim its d cells (a second key's claim marks the cell shared),
// fat_count_k / fat_emit_k write the shared pairs compacted in op order (a
// stable cell sort keeps each cell's ops in stream order) and each op's
// minimum over its exclusive rows into b_min, and fat_excl_final_k writes
// the exclusive cells' final values. The batch must be insert-only and
// free of saturation on exclusive cells (checked on the device, read once by
// the host; otherwise the batch takes the full sort).
template <int D>
struct FatArgs {
  KeySrc keys;
  const uint8_t* ops;
  uint32_t n;
  Seeds<D> seeds;
  Mod wm;
  uint32_t wp;
  const uint32_t* tb;       // key-sorted op list
  const uint32_t* headpos;  // [j]: position of j's key segment head
  const uint2* meta;        // [t]: {key count, previous op}
  uint32_t* owner;          // [cell]: the first key head that claimed it
  uint8_t* shared;          // [cell]: claimed by two or more keys
  const uint32_t* fat_init;
  uint32_t* fat;
  uint32_t* ncnt;           // [t]: the op's rows on shared cells (then their exclusive prefix sum)
  uint32_t* key_out;
  uint32_t* val_out;
  uint32_t* obs;            // [t]: min over the op's exclusive rows of its post-op count
  Ctl* ctl;
};

template <int D>
__global__ void __launch_bounds__(256) fat_owner_k(FatArgs<D> a) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < a.n; j += gridDim.x * blockDim.x) {
    if (a.headpos[j] != j) continue;
    const uint64_t key = load_key(a.keys, a.tb[j]);
#pragma unroll
    for (int i = 0; i < D; ++i) {
      const uint32_t f = (uint32_t)i * a.wp + (uint32_t)bucket(key, a.seeds.s[i], a.wm);
      const uint32_t prev = atomicCAS(a.owner + f, NONE32, j);
      if (prev != NONE32 && prev != j) a.shared[f] = 1;
    }
  }
}

template <int D>
__global__ void __launch_bounds__(256) fat_count_k(FatArgs<D> a) {
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < a.n; t += gridDim.x * blockDim.x) {
    const uint64_t key = load_key(a.keys, t);
    uint32_t c = 0;
#pragma unroll
    for (int i = 0; i < D; ++i) c += a.shared[(uint32_t)i * a.wp + (uint32_t)bucket(key, a.seeds.s[i], a.wm)];
    a.ncnt[t] = c;
  }
}

// (ncnt holds the exclusive prefix sums here: op t's first output slot)
template <int D>
__global__ void __launch_bounds__(256) fat_emit_k(FatArgs<D> a) {
  uint32_t local_fail = NONE32, local_bad = NONE32;
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < a.n; t += gridDim.x * blockDim.x) {
    const uint64_t key = load_key(a.keys, t);
    const uint32_t code = a.ops[t];
    const uint32_t op = code != 0;
    if (code > 1 && local_bad == NONE32) local_bad = t;
    if (op && local_fail == NONE32) local_fail = t;  // SF1: a delete is the failing op
    const uint64_t cnt = a.meta[t].x;
    uint32_t o = a.ncnt[t];
    uint64_t ex = ~0ull;
#pragma unroll
    for (int i = 0; i < D; ++i) {
      const uint32_t f = (uint32_t)i * a.wp + (uint32_t)bucket(key, a.seeds.s[i], a.wm);
      if (a.shared[f]) {
        a.key_out[o] = f;
        a.val_out[o] = (t << 1) | op;
        ++o;
      } else {
        const uint64_t post = (uint64_t)__ldg(a.fat_init + f) + cnt;
        if (post - 1 >= (uint64_t)U32MAX) local_fail = min(local_fail, t);  // a saturated counter before the op
        ex = min(ex, post);
      }
    }
    a.obs[t] = (uint32_t)min(ex, (uint64_t)U32MAX);
  }
  if (local_fail != NONE32) atomicMin(&a.ctl->fail_t, local_fail);
  if (local_bad != NONE32) {
    atomicMin(&a.ctl->bad_op, local_bad);
    atomicMin(&a.ctl->fail_t, 0u);
  }
}

// exclusive cells: the final value is the value before the batch plus the
// key's op count (the last op of a key segment carries it)
template <int D>
__global__ void __launch_bounds__(256) fat_excl_final_k(FatArgs<D> a) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < a.n; j += gridDim.x * blockDim.x) {
    if (j + 1 < a.n && a.headpos[j + 1] == a.headpos[j]) continue;  // not the segment's last op
    const uint32_t tot = j - a.headpos[j] + 1u;
    const uint64_t key = load_key(a.keys, a.tb[j]);
#pragma unroll
    for (int i = 0; i < D; ++i) {
      const uint32_t f = (uint32_t)i * a.wp + (uint32_t)bucket(key, a.seeds.s[i], a.wm);
      if (!a.shared[f]) a.fat[f] = a.fat_init[f] + tot;
    }
  }
}

int launch_load_keys(KeySrc ks, int64_t n, uint64_t* out, cudaStream_t st);  // sfk_query.cu

// per-op b_min from the fat scan's (t, candidate) pairs in k_in / v_in (see
// bmin_bucket_k); uses k_out / v_out (the fat-sorted pairs are dead by then).
// When t has more than 8 bits above BMIN_BITS, one 8-bit partial sort pass
// groups the pairs into 256 ranges of consecutive ops instead of two passes
// down to 2^BMIN_BITS, and the minima are taken with L2 atomics: CTAs walk
// the grouped pairs in order, so the ranges they update at any time (a few
// MB of b_min words) stay in L2 (cfg 4: one 400M-pair pass saved).
__global__ void __launch_bounds__(256) bmin_l2_k(const uint32_t* __restrict__ tkey, const uint32_t* __restrict__ tval,
                                                 uint32_t N, uint32_t* __restrict__ obs) {
  const uint32_t e0 = blockIdx.x * 2048u;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const uint32_t e = e0 + q * 256u + threadIdx.x;
    if (e < N) atomicMin(obs + __ldg(tkey + e), __ldg(tval + e));
  }
}
// compacted: the pairs cover only some of each op's rows (the shared-cell
// fat phase), and obs already holds the other rows' minimum
static int bmin_from_pairs(Layout& L, uint32_t n, uint32_t N, int d, cudaStream_t st, bool compacted = false) {
  const int tbits = bits_for((uint64_t)n);
  const uint32_t* tk = L.k_in;
  const uint32_t* tv = L.v_in;
  const bool l2 = compacted || tbits - BMIN_BITS > 8;
  if (tbits > BMIN_BITS) {
    size_t bytes = L.cub_tmp_bytes;
    cudaError_t e = cub::DeviceRadixSort::SortPairs(L.cub_tmp, bytes, L.k_in, L.k_out, L.v_in, L.v_out, (int)N,
                                                    l2 ? std::max(tbits - 8, 0) : BMIN_BITS, tbits, st);
    if (e != cudaSuccess) {
      set_error("b_min sort: %s", cudaGetErrorString(e));
      return (int)e;
    }
    tk = L.k_out;
    tv = L.v_out;
  }
  if (l2) {
    if (!compacted) cudaMemsetAsync(L.obs, 0xFF, (size_t)n * 4, st);
    { note_launch(); bmin_l2_k<<<(N + 2047) / 2048, 256, 0, st>>>(tk, tv, N, L.obs); }
    return check_launch("bmin_l2");
  }
  const uint32_t nb = (n + (1u << BMIN_BITS) - 1) >> BMIN_BITS;
  { note_launch(); bmin_bucket_k<<<nb, 512, 0, st>>>(tk, tv, n, (uint32_t)d, L.obs); }
  return check_launch("bmin_bucket");
}

// SF1 / CU key grouping: the key-sorted op list (tb), segment heads
// (headpos) and, per op, {key count, previous op of the key} (meta)
static int key_group(Layout& L, KeySrc ks, uint32_t n, cudaStream_t st, bool keys_loaded) {
  const int sms = sm_count();
  static const bool key_sort = getenv("SFK_KEY_GROUP") && !strcmp(getenv("SFK_KEY_GROUP"), "sort");  // A/B knob
  // u32 keys sort as they are (4 passes of 4-B keys); wider keys are materialised
  const bool direct32 = ks.kind == SFK_KEY_U32 && !key_sort;
  if (!keys_loaded && !direct32)
    if (int r = launch_load_keys(ks, n, L.k64a, st)) return r;
  { note_launch(); iota_k<<<grid_for(n, 256, sms * 8), 256, 0, st>>>(L.ta, n); }
  size_t bytes = L.cub_tmp_bytes;
  cudaError_t e;
  if (direct32) {
    uint32_t* sk = reinterpret_cast<uint32_t*>(L.k64b);  // the sorted keys
    e = cub::DeviceRadixSort::SortPairs(L.cub_tmp, bytes, static_cast<const uint32_t*>(ks.p), sk, L.ta, L.tb, (int)n,
                                        0, 32, st);
    if (e != cudaSuccess) { set_error("key sort: %s", cudaGetErrorString(e)); return (int)e; }
    { note_launch(); key_heads_k<uint32_t><<<grid_for(n, 256, sms * 8), 256, 0, st>>>(sk, n, L.headpos); }
    bytes = L.cub_tmp_bytes;
    e = cub::DeviceScan::InclusiveScan(L.cub_tmp, bytes, L.headpos, L.headpos, cub::Max(), (int)n, st);
    if (e != cudaSuccess) { set_error("key heads: %s", cudaGetErrorString(e)); return (int)e; }
    { note_launch(); key_meta_k<uint32_t><<<grid_for(n, 256, sms * 8), 256, 0, st>>>(sk, L.tb, L.headpos, n, L.meta); }
  } else if (ks.kind != SFK_KEY_U32 && !key_sort) {
    // 64-bit keys: group by table slot (4-B ids, see key_slot_k)
    const uint32_t cap = slot_cap(n);
    uint32_t* sid = reinterpret_cast<uint32_t*>(L.k64b);  // [0, n): ids in op order, [n, 2n): sorted
    cudaMemsetAsync(L.htab, 0xFF, (size_t)cap * 8, st);
    { note_launch(); key_slot_k<<<grid_for(n, 256, sms * 16), 256, 0, st>>>(L.k64a, n, L.htab, cap, sid); }
    e = cub::DeviceRadixSort::SortPairs(L.cub_tmp, bytes, sid, sid + n, L.ta, L.tb, (int)n, 0,
                                        bits_for((uint64_t)cap + 1), st);
    if (e != cudaSuccess) { set_error("key sort: %s", cudaGetErrorString(e)); return (int)e; }
    { note_launch(); key_heads_k<uint32_t><<<grid_for(n, 256, sms * 8), 256, 0, st>>>(sid + n, n, L.headpos); }
    bytes = L.cub_tmp_bytes;
    e = cub::DeviceScan::InclusiveScan(L.cub_tmp, bytes, L.headpos, L.headpos, cub::Max(), (int)n, st);
    if (e != cudaSuccess) { set_error("key heads: %s", cudaGetErrorString(e)); return (int)e; }
    { note_launch(); key_meta_k<uint32_t><<<grid_for(n, 256, sms * 8), 256, 0, st>>>(sid + n, L.tb, L.headpos, n, L.meta); }
  } else {
    const int kbits = ks.kind == SFK_KEY_U32 ? 32 : 64;
    e = cub::DeviceRadixSort::SortPairs(L.cub_tmp, bytes, L.k64a, L.k64b, L.ta, L.tb, (int)n, 0, kbits, st);
    if (e != cudaSuccess) { set_error("key sort: %s", cudaGetErrorString(e)); return (int)e; }
    { note_launch(); key_heads_k<uint64_t><<<grid_for(n, 256, sms * 8), 256, 0, st>>>(L.k64b, n, L.headpos); }
    bytes = L.cub_tmp_bytes;
    e = cub::DeviceScan::InclusiveScan(L.cub_tmp, bytes, L.headpos, L.headpos, cub::Max(), (int)n, st);
    if (e != cudaSuccess) { set_error("key heads: %s", cudaGetErrorString(e)); return (int)e; }
    { note_launch(); key_meta_k<uint64_t><<<grid_for(n, 256, sms * 8), 256, 0, st>>>(L.k64b, L.tb, L.headpos, n, L.meta); }
  }
  return 0;
}

// SF1: per-op key counts (sort by key), dropped (op, row) flags, filtered links
static int sf1_ignore_pass(Layout& L, KeySrc ks, uint32_t n, uint32_t N, uint32_t w, uint32_t D, cudaStream_t st,
                           bool keys_loaded = false, bool grouped = false, bool bmin_by_pos = false) {
  const int sms = sm_count();
  cudaError_t e;
  if (!grouped)
    if (int r = key_group(L, ks, n, st, keys_loaded)) return r;
  const uint32_t ntiles = (N + SCAN_TILE - 1) / SCAN_TILE;
  // {key count, b_min, previous op} per op, gathered once by the ignore scan
  // in cell order; 16 n bytes over k64a and k64b (adjacent, dead after the
  // key grouping)
  if (reinterpret_cast<char*>(L.k64b) < reinterpret_cast<char*>(L.k64a) ||
      reinterpret_cast<char*>(L.k64a) + 16ull * n > reinterpret_cast<char*>(L.k64b) + 8ull * n) {
    set_error("workspace layout: k64a and k64b must be adjacent");  // (carve() keeps them so)
    return 1;
  }
  uint4* cb = reinterpret_cast<uint4*>(L.k64a);
  uint32_t* kpc = L.v_in;  // the previous op per element in cell order (v_in is dead after the slim sort)
  cudaMemsetAsync(L.dmask, 0, ((size_t)n / 4 + 1) * 4, st);
  cudaMemsetAsync(L.rbrk, 0, ((size_t)n / 32 + 1) * 4, st);
  cudaMemsetAsync(L.hbitsj, 0, ((size_t)n / 32 + 1) * 4, st);
  { note_launch(); cb_pack_k<<<grid_for(n, 256, sms * 8), 256, 0, st>>>(L.tb, L.headpos, L.obs, bmin_by_pos ? 1 : 0, n, cb); }
  { note_launch(); sf1_ignore_k<<<ntiles, SCAN_THREADS, 0, st>>>(L.k_out, L.v_out, N, w, cb, L.ctl, L.ign, kpc, L.dmask); }
  // ftiles: [tile aggregates][their exclusive prefixes][scan temp storage]
  SegCnt* ft = static_cast<SegCnt*>(L.ftiles);
  SegCnt* fc = ft + ntiles;
  void* ftmp = reinterpret_cast<void*>((reinterpret_cast<uintptr_t>(fc + ntiles) + 255) & ~uintptr_t(255));
  { note_launch(); filt_reduce_k<<<ntiles, SCAN_THREADS, 0, st>>>(L.k_out, L.v_out, L.ign, N, ft); }
  size_t fbytes = 0;
  cub::DeviceScan::ExclusiveScan(nullptr, fbytes, ft, fc, SegCntOp(), SegCnt{0u, 0u, NONE32}, (int)ntiles, st);
  e = cub::DeviceScan::ExclusiveScan(ftmp, fbytes, ft, fc, SegCntOp(), SegCnt{0u, 0u, NONE32}, (int)ntiles, st);
  if (e != cudaSuccess) { set_error("filtered-link tiles: %s", cudaGetErrorString(e)); return (int)e; }
  { note_launch(); filt_apply_k<false><<<ntiles, SCAN_THREADS, 0, st>>>(L.k_out, L.v_out, L.ign, N, D, w, fc, kpc, L.tb, L.rbrk, nullptr); }
  { note_launch(); runs_head_ign_k<<<grid_for(n, 256, sms * 16), 256, 0, st>>>(n, L.ctl, reinterpret_cast<const uint8_t*>(L.dmask), L.rbrk, L.meta, D, L.headflag, L.hbits, L.hbitsj); }
  { note_launch(); filt_apply_k<true><<<ntiles, SCAN_THREADS, 0, st>>>(L.k_out, L.v_out, L.ign, N, D, w, fc, nullptr, L.tb, L.hbitsj, reinterpret_cast<uint4*>(L.links)); }
  return check_launch("sf1_ignore");
}

template <int D>
static int sf_parallel_d(int kind, uint32_t* slim, uint32_t* fat, uint32_t* dsub, const uint64_t* slim_seeds,
                         const uint64_t* fat_seeds, int64_t w, int64_t wp, int z, const uint8_t* ops, KeySrc ks,
                         int64_t n64, int64_t* inc, int64_t* result, Layout& L, cudaStream_t st, const ExtArgs* ext) {
  const int sms = sm_count();
  const uint32_t n = (uint32_t)n64;
  const uint32_t N = (uint32_t)(D * n64);
  { note_launch(); ctl_init_k<<<1, 1, 0, st>>>(L.ctl); }
  if (kind == 0) {  // ------------------------------------------------ SFF
    const int kb = bits_for((uint64_t)z);
    HashArgs<D> h = make_hash<D>(ks, ops, n64, slim_seeds, fat_seeds, (uint64_t)w, z, kb, L, 0);
    { note_launch(); hash_emit_k<D, 0><<<grid_for(n64, 256, sms * 16), 256, 0, st>>>(h); }
    if (int r = sort_pairs(L, N, D, (uint64_t)w, st)) return r;
    const size_t fat_bytes = (size_t)D * w * z * 4;
    cudaMemcpyAsync(L.fat_snap, fat, fat_bytes, cudaMemcpyDeviceToDevice, st);
    ScanOut so{L.fat_snap, fat, nullptr, L.obs2, L.links, n, (uint32_t)D, (uint32_t)w, L.ctl};
    if (int r = run_scan_z<true, 2, true>(z, L.k_out, L.v_out, N, kb, L.tiles, so, st)) return r;
    { note_launch(); fat_undo_k<D, 0><<<grid_for(n64, 256, sms * 8), 256, 0, st>>>(h, fat, (uint32_t)z); }
    if (int r = run_engine<D, 2>(L, slim, slim_seeds, w, ks, n, kb, inc, st)) return r;
    { note_launch(); finalize_k<<<1, 1, 0, st>>>(L.ctl, ops, 1, result, nullptr, D, 0); }
  } else if (kind == 1) {  // ------------------------------------------ SF1
    // record keys (FNV-1a + finalize64 over 13 B) are hashed once into k64a
    // and read back as u64 by the hash emits and the key grouping
    const bool ign = D > 1 && !getenv("SFK_NO_SF1_IGNORE");  // diagnostics knob
    const bool mat = ign && ks.kind == SFK_KEY_RECORD;
    if (mat)
      if (int r = launch_load_keys(ks, n64, L.k64a, st)) return r;
    const KeySrc kh = mat ? KeySrc{L.k64a, SFK_KEY_U64, 8} : ks;
    HashArgs<D> hf = make_hash<D>(kh, ops, n64, fat_seeds, nullptr, (uint64_t)wp, 1, 0, L, 1);
    cudaMemcpyAsync(L.fat_snap, fat, (size_t)D * wp * 4, cudaMemcpyDeviceToDevice, st);
    // large batches: the fat sort and scan only over pairs on shared cells
    // (fat_owner_k ...); one host read of {pairs, t*}. Not while the stream
    // is being captured into a graph (no host read there), and not for
    // batches that fail (deletes, saturation): those take the full sort.
    static const bool fat_sort = getenv("SFK_SF1_FAT") && !strcmp(getenv("SFK_SF1_FAT"), "sort");  // A/B knob
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cap);
    const char* fmin = getenv("SFK_SF1_FAT_MIN");  // tests: smallest batch for this path (default 2^20 ops)
    const uint32_t excl_min = fmin ? (uint32_t)strtoul(fmin, nullptr, 10) : (1u << 20);
    bool grouped = false, excl = ign && !fat_sort && n >= excl_min && cap == cudaStreamCaptureStatusNone;
    if (excl) {
      if (int r = key_group(L, kh, n, st, mat)) return r;
      grouped = true;
      FatArgs<D> fa;
      fa.keys = kh;
      fa.ops = ops;
      fa.n = n;
      for (int i = 0; i < D; ++i) fa.seeds.s[i] = fat_seeds[i];
      fa.wm = make_mod((uint64_t)wp);
      fa.wp = (uint32_t)wp;
      fa.tb = L.tb;
      fa.headpos = L.headpos;
      fa.meta = L.meta;
      fa.owner = L.owner;
      fa.shared = L.shared;
      fa.fat_init = L.fat_snap;
      fa.fat = fat;
      fa.ncnt = L.ncnt;
      fa.key_out = L.k_in;
      fa.val_out = L.v_in;
      fa.obs = L.obs;
      fa.ctl = L.ctl;
      cudaMemsetAsync(L.owner, 0xFF, (size_t)D * wp * 4, st);
      cudaMemsetAsync(L.shared, 0, (size_t)D * wp, st);
      cudaMemsetAsync(L.ncnt + n, 0, 4, st);
      { note_launch(); fat_owner_k<D><<<grid_for(n64, 256, sms * 8), 256, 0, st>>>(fa); }
      { note_launch(); fat_count_k<D><<<grid_for(n64, 256, sms * 8), 256, 0, st>>>(fa); }
      size_t bytes = L.cub_tmp_bytes;
      if (cub::DeviceScan::ExclusiveSum(L.cub_tmp, bytes, L.ncnt, L.noff, (int)n + 1, st) != cudaSuccess) {
        set_error("shared-pair offsets: scan failed");
        return 1;
      }
      fa.ncnt = L.noff;
      { note_launch(); fat_emit_k<D><<<grid_for(n64, 256, sms * 8), 256, 0, st>>>(fa); }
      uint32_t hv[2];
      cudaMemcpyAsync(hv, L.noff + n, 4, cudaMemcpyDeviceToHost, st);
      cudaMemcpyAsync(hv + 1, &L.ctl->fail_t, 4, cudaMemcpyDeviceToHost, st);
      if (cudaStreamSynchronize(st) != cudaSuccess) return check_launch("shared-pair count");
      if (hv[1] != NONE32) {  // a delete, a bad op code or a saturated exclusive cell: the full sort
        excl = false;
        { note_launch(); ctl_init_k<<<1, 1, 0, st>>>(L.ctl); }
      } else {
        const uint32_t Ns = hv[0];
        { note_launch(); fat_excl_final_k<D><<<grid_for(n64, 256, sms * 8), 256, 0, st>>>(fa); }
        if (Ns) {
          bytes = L.cub_tmp_bytes;
          if (cub::DeviceRadixSort::SortPairs(L.cub_tmp, bytes, L.k_in, L.k_out, L.v_in, L.v_out, (int)Ns, 0,
                                              std::max(bits_for((uint64_t)D * wp), 1), st) != cudaSuccess) {
            set_error("shared-pair sort failed");
            return 1;
          }
          ScanOut sf{L.fat_snap, fat, L.obs, nullptr, nullptr, n, (uint32_t)D, (uint32_t)wp, L.ctl, L.k_in, L.v_in};
          if (int r = run_scan_z<true, 6, false>(1, L.k_out, L.v_out, Ns, 0, L.tiles, sf, st)) return r;
          if (int r = bmin_from_pairs(L, n, Ns, D, st, true)) return r;
        }
      }
    }
    if (!excl) {
      { note_launch(); hash_emit_k<D, 1><<<grid_for(n64, 256, sms * 16), 256, 0, st>>>(hf); }
      if (int r = sort_pairs(L, N, D, (uint64_t)wp, st)) return r;
      ScanOut sf{L.fat_snap, fat, L.obs, nullptr, nullptr, n, (uint32_t)D, (uint32_t)wp, L.ctl, L.k_in, L.v_in};
      if (int r = run_scan_z<true, 6, false>(1, L.k_out, L.v_out, N, 0, L.tiles, sf, st)) return r;
      if (int r = bmin_from_pairs(L, n, N, D, st)) return r;
    }
    { note_launch(); fat_undo_k<D, 1><<<grid_for(n64, 256, sms * 8), 256, 0, st>>>(hf, fat, 1u); }
    HashArgs<D> hs = make_hash<D>(kh, ops, n64, slim_seeds, nullptr, (uint64_t)w, 1, 0, L, 0);
    if (ign) {  // slim pairs name their ops by key-order position (key_meta_k)
      if (!grouped)
        if (int r = key_group(L, kh, n, st, mat)) return r;
      grouped = true;
      hs.pos = L.meta;
    }
    { note_launch(); hash_emit_k<D, 2><<<grid_for(n64, 256, sms * 16), 256, 0, st>>>(hs); }
    if (int r = sort_pairs(L, N, D, (uint64_t)w, st)) return r;
    if (ign) {  // the filtered scan writes the run heads' link records itself
      if (int r = sf1_ignore_pass(L, ks, n, N, (uint32_t)w, (uint32_t)D, st, mat, grouped)) return r;
    } else {
      ScanOut ss{nullptr, nullptr, nullptr, nullptr, L.links, n, (uint32_t)D, (uint32_t)w, L.ctl};
      if (int r = run_scan_z<false, 0, true>(1, L.k_out, L.v_out, N, 0, L.tiles, ss, st)) return r;
    }
    if (int r = run_engine<D, 0>(L, slim, slim_seeds, w, ks, n, 0, inc, st, false, ign)) return r;
    { note_launch(); finalize_k<<<1, 1, 0, st>>>(L.ctl, ops, 0, result, nullptr, D, 0); }
  } else if (kind == 4 || kind == 5) {  // -------------------------- SF4 / SF3
    // SF4: buckets by the slim seeds, slots by the extended seeds (as SFF).
    // SF3: g = h_i(key) over w' = z w (slim seeds), bucket g mod w, slot g / w.
    const int kb = bits_for((uint64_t)z);
    const bool fold = kind == 5;
    HashArgs<D> h = fold ? make_hash<D>(ks, ops, n64, slim_seeds, nullptr, (uint64_t)wp, z, kb, L, 0)
                         : make_hash<D>(ks, ops, n64, slim_seeds, fat_seeds, (uint64_t)w, z, kb, L, 0);
    h.fold_w = (uint32_t)w;
    if (fold) { note_launch(); hash_emit_k<D, 3><<<grid_for(n64, 256, sms * 16), 256, 0, st>>>(h); }
    else { note_launch(); hash_emit_k<D, 0><<<grid_for(n64, 256, sms * 16), 256, 0, st>>>(h); }
    if (int r = sort_pairs(L, N, D, (uint64_t)w, st)) return r;
    const uint64_t cells = (uint64_t)D * w * z;
    uint32_t* fat_grp = fat;
    if (fold) {
      { note_launch(); fold_gather_k<<<grid_for((int64_t)cells, 256, sms * 8), 256, 0, st>>>(fat, L.fat_snap, D, (uint32_t)w, (uint32_t)z); }
      // the scan writes only the groups this batch touches
      cudaMemcpyAsync(L.fat_perm, L.fat_snap, cells * 4, cudaMemcpyDeviceToDevice, st);
      fat_grp = L.fat_perm;
    } else {
      cudaMemcpyAsync(L.fat_snap, fat, cells * 4, cudaMemcpyDeviceToDevice, st);
    }
    ScanOut so{L.fat_snap, fat_grp, nullptr, L.obs2, L.links, n, (uint32_t)D, (uint32_t)w, L.ctl};
    if (int r = run_scan_z<true, 3, true>(z, L.k_out, L.v_out, N, kb, L.tiles, so, st)) return r;
    if (fold) {
      { note_launch(); fold_scatter_k<<<grid_for((int64_t)cells, 256, sms * 8), 256, 0, st>>>(L.fat_perm, fat, D, (uint32_t)w, (uint32_t)z); }
      HashArgs<D> hf = make_hash<D>(ks, ops, n64, slim_seeds, nullptr, (uint64_t)wp, 1, 0, L, 0);
      { note_launch(); fat_undo_k<D, 1><<<grid_for(n64, 256, sms * 8), 256, 0, st>>>(hf, fat, 1u); }
    } else {
      { note_launch(); fat_undo_k<D, 0><<<grid_for(n64, 256, sms * 8), 256, 0, st>>>(h, fat, (uint32_t)z); }
    }
    if (int r = run_engine<D, 3>(L, slim, slim_seeds, w, ks, n, kb, inc, st)) return r;
    { note_launch(); finalize_k<<<1, 1, 0, st>>>(L.ctl, ops, 1, result, nullptr, D, 0); }
  } else if (kind == 6) {  // ------------------------------------------ SF2
    // flat fat: per-op b_min (as SF1, deletes allowed); deletion sub-sketch on
    // the slim cells: a second, slim-sorted scan carries its counts
    HashArgs<D> hf = make_hash<D>(ks, ops, n64, fat_seeds, nullptr, (uint64_t)wp, 1, 0, L, 0);
    { note_launch(); hash_emit_k<D, 1><<<grid_for(n64, 256, sms * 16), 256, 0, st>>>(hf); }
    if (int r = sort_pairs(L, N, D, (uint64_t)wp, st)) return r;
    cudaMemcpyAsync(L.fat_snap, fat, (size_t)D * wp * 4, cudaMemcpyDeviceToDevice, st);
    ScanOut sf{L.fat_snap, fat, L.obs, nullptr, nullptr, n, (uint32_t)D, (uint32_t)wp, L.ctl, L.k_in, L.v_in};
    if (int r = run_scan_z<true, 6, false>(1, L.k_out, L.v_out, N, 0, L.tiles, sf, st)) return r;
    if (int r = bmin_from_pairs(L, n, N, D, st)) return r;
    HashArgs<D> hs = make_hash<D>(ks, ops, n64, slim_seeds, nullptr, (uint64_t)w, 1, 0, L, 0);
    { note_launch(); hash_emit_k<D, 2><<<grid_for(n64, 256, sms * 16), 256, 0, st>>>(hs); }
    if (int r = sort_pairs(L, N, D, (uint64_t)w, st)) return r;
    cudaMemcpyAsync(L.fat_snap, dsub, (size_t)D * w * 4, cudaMemcpyDeviceToDevice, st);
    ScanOut sd{L.fat_snap, dsub, nullptr, L.obs2, L.links, n, (uint32_t)D, (uint32_t)w, L.ctl};
    if (int r = run_scan_z<true, 3, true>(1, L.k_out, L.v_out, N, 0, L.tiles, sd, st)) return r;
    // both scans can find the failing op (the deletion sub-sketch its own
    // phantom / saturation): undo both only once t* is final
    { note_launch(); fat_undo_k<D, 1><<<grid_for(n64, 256, sms * 8), 256, 0, st>>>(hf, fat, 1u); }
    { note_launch(); fat_undo_k<D, 2><<<grid_for(n64, 256, sms * 8), 256, 0, st>>>(hs, dsub, 1u); }
    if (int r = run_engine<D, 3>(L, slim, slim_seeds, w, ks, n, 0, inc, st, true)) return r;
    { note_launch(); finalize_k<<<1, 1, 0, st>>>(L.ctl, ops, 1, result, nullptr, D, 0); }
  } else if (kind == 7 || kind == 8) {  // ----------------- CML / oracle-assisted
    // insert-only gated min-raise on the slim-shaped table with a per-op
    // cap (the CML coin flip as an exponent bound, or the true count); the
    // cap is not monotone along a run, so runs replay op by op (MODE 3 with
    // per-op data)
    const uint32_t cells = (uint32_t)(D * w);
    uint32_t* tab = slim;
    const uint8_t* opk = ops;
    if (kind == 7) {
      { note_launch(); widen_u16_k<<<grid_for(cells, 256, sms * 8), 256, 0, st>>>(ext->exps, L.fat_snap, cells); }
      tab = L.fat_snap;
    } else {
      cudaMemsetAsync(L.zops, 0, (size_t)n64, st);
      opk = L.zops;
    }
    HashArgs<D> hs = make_hash<D>(ks, opk, n64, slim_seeds, nullptr, (uint64_t)w, 1, 0, L, 1);
    { note_launch(); hash_emit_k<D, 2><<<grid_for(n64, 256, sms * 16), 256, 0, st>>>(hs); }
    if (int r = sort_pairs(L, N, D, (uint64_t)w, st)) return r;
    ScanOut ss{nullptr, nullptr, nullptr, nullptr, L.links, n, (uint32_t)D, (uint32_t)w, L.ctl};
    if (int r = run_scan_z<false, 0, true>(1, L.k_out, L.v_out, N, 0, L.tiles, ss, st)) return r;
    if (kind == 7) { note_launch(); cml_gate_k<<<grid_for(n64, 256, sms * 8), 256, 0, st>>>(ext->gate, ext->rng_seed, ext->start_pos, n, L.obs); }
    else { note_launch(); oracle_gate_k<<<grid_for(n64, 256, sms * 8), 256, 0, st>>>(ext->true_counts, n, L.obs); }
    if (int r = run_engine<D, 3>(L, tab, slim_seeds, w, ks, n, 0, kind == 7 ? L.inc_scratch : inc, st, true, false,
                                 true, kind == 8))
      return r;
    if (kind == 7) { note_launch(); narrow_u16_k<<<grid_for(cells, 256, sms * 8), 256, 0, st>>>(L.fat_snap, ext->exps, cells); }
    { note_launch(); finalize_k<<<1, 1, 0, st>>>(L.ctl, opk, 0, result, nullptr, D, 0); }
  } else if (kind == 2) {  // ------------------------------------------ CU
    HashArgs<D> hs = make_hash<D>(ks, ops, n64, slim_seeds, nullptr, (uint64_t)w, 1, 0, L, 1);
    const bool ign = D > 1 && !getenv("SFK_NO_SF1_IGNORE");  // diagnostics knob (shared with SF1)
    if (ign) {  // slim pairs name their ops by key-order position (key_meta_k)
      if (int r = key_group(L, ks, n, st, false)) return r;
      hs.pos = L.meta;
    }
    { note_launch(); hash_emit_k<D, 2><<<grid_for(n64, 256, sms * 16), 256, 0, st>>>(hs); }
    if (int r = sort_pairs(L, N, D, (uint64_t)w, st)) return r;
    if (!ign) {
      ScanOut ss{nullptr, nullptr, nullptr, nullptr, L.links, n, (uint32_t)D, (uint32_t)w, L.ctl};
      if (int r = run_scan_z<false, 0, true>(1, L.k_out, L.v_out, N, 0, L.tiles, ss, st)) return r;
    } else {  // the filtered scan writes every link record itself
      // a CU cell is >= the batch count of every key on it, and <= its value
      // before the batch + the ops on it so far: an op drops the rows whose
      // lower bound exceeds that upper bound of its own minimum
      ScanOut su{slim, nullptr, L.obs, nullptr, nullptr, n, (uint32_t)D, (uint32_t)w, L.ctl};
      cudaMemsetAsync(L.obs, 0xFF, (size_t)n * 4, st);
      if (int r = run_scan<1, false, 5, false>(L.k_out, L.v_out, N, 0, L.tiles, su, st)) return r;
      if (int r = sf1_ignore_pass(L, ks, n, N, (uint32_t)w, (uint32_t)D, st, false, true, true)) return r;
    }
    if (int r = run_engine<D, 1>(L, slim, slim_seeds, w, ks, n, 0, inc, st, false, ign)) return r;
    { note_launch(); finalize_k<<<1, 1, 0, st>>>(L.ctl, ops, 0, result, nullptr, D, 0); }
  } else {  // ------------------------------------------------------- CM exact
    HashArgs<D> h = make_hash<D>(ks, ops, n64, slim_seeds, nullptr, (uint64_t)w, 1, 0, L, 0);
    { note_launch(); hash_emit_k<D, 2><<<grid_for(n64, 256, sms * 16), 256, 0, st>>>(h); }
    if (int r = sort_pairs(L, N, D, (uint64_t)w, st)) return r;
    cudaMemcpyAsync(L.fat_snap, slim, (size_t)D * w * 4, cudaMemcpyDeviceToDevice, st);
    ScanOut so{L.fat_snap, slim, nullptr, nullptr, nullptr, n, (uint32_t)D, (uint32_t)w, L.ctl};
    if (int r = run_scan_z<true, 0, false>(1, L.k_out, L.v_out, N, 0, L.tiles, so, st)) return r;
    { note_launch(); fat_undo_k<D, 2><<<grid_for(n64, 256, sms * 8), 256, 0, st>>>(h, slim, 1u); }
    { note_launch(); count_ins_k<<<grid_for(n64, 256, sms * 8), 256, 0, st>>>(ops, n64, L.ctl); }
    { note_launch(); finalize_k<<<1, 1, 0, st>>>(L.ctl, ops, 1, result, reinterpret_cast<unsigned long long*>(inc), D, 1); }
  }
  return check_launch("sf_parallel");
}

int parallel_apply(int kind, uint32_t* slim, uint32_t* fat, uint32_t* dsub, const uint64_t* slim_seeds,
                   const uint64_t* fat_seeds, int d, int64_t w, int64_t wp, int z, const uint8_t* ops, KeySrc ks,
                   int64_t n, int64_t* inc, int64_t* result, void* ws, size_t ws_bytes, cudaStream_t st,
                   const ExtArgs* ext) {
  Layout L = carve(ws, ws_bytes, kind, d, w, wp, z, n);
  if (!L.ok || ws == nullptr) {
    set_error("workspace too small: need %zu bytes, got %zu", L.total, ws_bytes);
    return 1;
  }
  if ((kind == 7 || kind == 8) && ext == nullptr) {
    set_error("gated engine kind %d needs its per-op gate arguments", kind);
    return 1;
  }
  switch (d) {
    case 1: return sf_parallel_d<1>(kind, slim, fat, dsub, slim_seeds, fat_seeds, w, wp, z, ops, ks, n, inc, result, L, st, ext);
    case 2: return sf_parallel_d<2>(kind, slim, fat, dsub, slim_seeds, fat_seeds, w, wp, z, ops, ks, n, inc, result, L, st, ext);
    case 3: return sf_parallel_d<3>(kind, slim, fat, dsub, slim_seeds, fat_seeds, w, wp, z, ops, ks, n, inc, result, L, st, ext);
    case 4: return sf_parallel_d<4>(kind, slim, fat, dsub, slim_seeds, fat_seeds, w, wp, z, ops, ks, n, inc, result, L, st, ext);
    case 5: return sf_parallel_d<5>(kind, slim, fat, dsub, slim_seeds, fat_seeds, w, wp, z, ops, ks, n, inc, result, L, st, ext);
    case 6: return sf_parallel_d<6>(kind, slim, fat, dsub, slim_seeds, fat_seeds, w, wp, z, ops, ks, n, inc, result, L, st, ext);
    case 7: return sf_parallel_d<7>(kind, slim, fat, dsub, slim_seeds, fat_seeds, w, wp, z, ops, ks, n, inc, result, L, st, ext);
    case 8: return sf_parallel_d<8>(kind, slim, fat, dsub, slim_seeds, fat_seeds, w, wp, z, ops, ks, n, inc, result, L, st, ext);
  }
  set_error("parallel engine: unsupported d=%d", d);
  return 1;
}

// CM/CU precheck statistics (host reads them back: one small sync)
int collect_stats(const uint8_t* ops, int64_t n, const uint32_t* counters, int64_t cells, void* ws, size_t ws_bytes,
                  Stats* host, cudaStream_t st, uint32_t bias) {
  Carver cv(ws, ws_bytes);
  cv.take<Ctl>(1);
  Stats* s = cv.take<Stats>(1);
  Stats init{};
  init.first_del = (unsigned long long)n;
  init.first_bad = (unsigned long long)n;
  init.cmax = 0;
  init.cmin = U32MAX;
  cudaMemcpyAsync(s, &init, sizeof(Stats), cudaMemcpyHostToDevice, st);
  const int sms = sm_count();
  if (n > 0) { note_launch(); stats_ops_k<<<grid_for(n, 256, sms * 8), 256, 0, st>>>(ops, n, s); }
  if (n > 0) { note_launch(); stats_ins_before_k<<<grid_for(n, 256, sms * 8), 256, 0, st>>>(ops, s); }
  { note_launch(); stats_counters_k<<<grid_for(cells, 256, sms * 8), 256, 0, st>>>(counters, cells, s, bias); }
  cudaMemcpyAsync(host, s, sizeof(Stats), cudaMemcpyDeviceToHost, st);
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    set_error("stats: %s", cudaGetErrorString(e));
    return (int)e;
  }
  return 0;
}

template <int D>
static int cm_fast_d(uint32_t* counters, const uint64_t* seeds, int64_t w, const uint8_t* ops, KeySrc ks, int64_t n,
                     cudaStream_t st) {
  Seeds<D> sd;
  for (int i = 0; i < D; ++i) sd.s[i] = seeds[i];
  const int sms = sm_count();
  { note_launch(); cm_atomic_k<D><<<grid_for((n + 31) / 32 * 32, 256, sms * 16), 256, 0, st>>>(counters, sd, make_mod((uint64_t)w),
                                                                              (uint32_t)w, ops, ks, n, nullptr); }
  return check_launch("cm_atomic");
}

int cm_fast(uint32_t* counters, const uint64_t* seeds, int d, int64_t w, const uint8_t* ops, KeySrc ks, int64_t n,
            cudaStream_t st) {
  switch (d) {
    case 1: return cm_fast_d<1>(counters, seeds, w, ops, ks, n, st);
    case 2: return cm_fast_d<2>(counters, seeds, w, ops, ks, n, st);
    case 3: return cm_fast_d<3>(counters, seeds, w, ops, ks, n, st);
    case 4: return cm_fast_d<4>(counters, seeds, w, ops, ks, n, st);
    case 5: return cm_fast_d<5>(counters, seeds, w, ops, ks, n, st);
    case 6: return cm_fast_d<6>(counters, seeds, w, ops, ks, n, st);
    case 7: return cm_fast_d<7>(counters, seeds, w, ops, ks, n, st);
    case 8: return cm_fast_d<8>(counters, seeds, w, ops, ks, n, st);
  }
  set_error("cm fast path: unsupported d=%d", d);
  return 1;
}

}  // namespace sfk
