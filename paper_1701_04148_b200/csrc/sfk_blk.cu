// Block engine: one 1024-thread CTA applies a whole medium SFF / SF4 batch
// (a few hundred to a few thousand ops, up to BLK_N (op, row) pairs) exactly,
// in one launch and in shared memory. It is the parallel pipeline of
// sfk_sf.cu folded into one CTA for the batches whose cost that pipeline's
// ~20 launches dominate (~150 us for 1K ops): the reference applies
// sf_bucket_apply (_kernels.py:318-384) op by op, and a 1K-op batch is ~50 us
// of one CPU thread there.
//   1. hash every (op, row) to its slim cell and fat slot; block radix sort
//      of the (cell, t | slot) pairs (stable: per cell in stream order);
//   2. a block-wide segmented scan over the sorted pairs carries each
//      cell's per-slot counts: per (op, row) the observation the slim update
//      needs (the own slot count after an insert; the bucket's max / sum
//      after a delete), its rank in the cell's sequence, the first failing
//      op; each cell's last pair writes the bucket back;
//   3. dataflow replay: the warp that owns op t's row-0 cell (so a key's ops
//      stay in one warp, in stream order, lane i on row i) applies it once
//      every cell of the op has applied the op's predecessors (per-cell
//      sequence counters in shared memory; a cell the warp touched last is
//      current in a register), exactly as the reference: m = min of the d cells,
//      b_min = min of the own slot counts, raise the cells at m if m < b_min;
//      a delete clamps to the bucket max (SFF) or steps down when above the
//      bucket sum (SF4);
//   4. write back slim cells, tallies and the result triple (a failing op
//      takes its and the later ops' fat deltas back).
#include <cub/block/block_radix_sort.cuh>

#include "../../include/sfsketch_cuda.h"
#include "sfk_common.cuh"

namespace sfk {

constexpr int BLK_T = 1024, BLK_IPT = 8, BLK_N = BLK_T * BLK_IPT;  // (op, row) pairs per batch
constexpr int BLK_ZMAX = 8;   // fat slots per bucket (the scan carries one count per slot)
template <int IPT>
using BlkSort = cub::BlockRadixSort<uint32_t, BLK_T, IPT, uint32_t>;

struct BlkArgs {
  uint32_t* slim;
  uint32_t* fat;
  Seeds<MAXD> s_seeds, f_seeds;
  int d, z, n, variant;  // variant 1: SFF (max clamp), 0: SF4 (sum trigger)
  int64_t w;
  Mod wm, zm;
  int kbits;              // sort bits: cells d * w
  const uint8_t* ops;
  KeySrc keys;
  int64_t* inc;
  int64_t* result;
};

// segmented-scan state over the sorted pairs: a cell starts in the span
// (flag), the position of the last such start (head), per-slot net counts
// since it (or over the span)
template <int Z>
struct BState {
  uint32_t flag, head;
  uint32_t v[Z];  // mod 2^32
};
template <int Z>
struct BStateOp {
  __device__ __forceinline__ BState<Z> operator()(const BState<Z>& a, const BState<Z>& b) const {
    if (b.flag) return b;
    BState<Z> r;
    r.flag = a.flag;
    r.head = a.head;
#pragma unroll
    for (int k = 0; k < Z; ++k) r.v[k] = a.v[k] + b.v[k];
    return r;
  }
};

__host__ __device__ constexpr size_t blk_align(size_t x) { return (x + 15) & ~size_t(15); }
__host__ __device__ constexpr size_t blk_max(size_t a, size_t b) { return a > b ? a : b; }

// shared memory: [sort / scan temp, then obs][sk][sv][seg][rnk][sl][sq][ops]
template <int Z>
struct BlkSmem {
  static constexpr size_t tmp = 0;
  static constexpr size_t obs = 0;                 // per (op, row), index t * d + i (after the scan)
  static constexpr size_t sk = blk_align(blk_max(blk_max(sizeof(typename BlkSort<BLK_IPT>::TempStorage),
                                                         sizeof(typename cub::BlockScan<BState<Z>, BLK_T>::TempStorage)),
                                                 (size_t)BLK_N * 4));
  static constexpr size_t sv = sk + BLK_N * 4;     // the sorted pair values
  static constexpr size_t seg = sv + BLK_N * 4;    // per (op, row): the sorted position of the cell's first pair
  static constexpr size_t rnk = seg + BLK_N * 2;   //   the pair's rank in its cell's sequence
  static constexpr size_t sl = rnk + BLK_N * 2;    // per cell (at its first pair's position): slim value
  static constexpr size_t sq = sl + BLK_N * 4;     //   and how many of its ops were applied
  static constexpr size_t ops = sq + BLK_N * 2;    // per op: its code (0 insert / 1 delete)
  static constexpr size_t total = ops + BLK_N;
};
static_assert(BlkSmem<8>::total <= 227 * 1024, "block engine shared memory");

// diagnostics: globaltimer at the phase boundaries of the last launch (ns)
__device__ unsigned long long g_blk_prof[8];
__device__ __forceinline__ void blk_stamp(int k) {
  if (threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_blk_prof[k] = t;
  }
}

__device__ __forceinline__ uint32_t ld_acq16(const uint16_t* p) {
  uint16_t v;
  asm volatile("ld.acquire.cta.shared::cta.u16 %0, [%1];" : "=h"(v) : "r"((uint32_t)__cvta_generic_to_shared(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel16(uint16_t* p, uint32_t v) {
  asm volatile("st.release.cta.shared::cta.u16 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(p)), "h"((uint16_t)v)
               : "memory");
}

// sorted pair value: t << 8 | row << 4 | op << 3 | slot (t < 8192, row < 8, slot < 8)
// IPT: pairs per thread in the sort and scan (N <= 1024 IPT)
template <int Z, int IPT>
__global__ void __launch_bounds__(BLK_T, 1) blk_bucket_k(BlkArgs a) {
  using S = BlkSmem<Z>;
  extern __shared__ __align__(16) unsigned char sm[];
  uint32_t* sk = reinterpret_cast<uint32_t*>(sm + S::sk);
  uint32_t* sv = reinterpret_cast<uint32_t*>(sm + S::sv);
  uint32_t* obs = reinterpret_cast<uint32_t*>(sm + S::obs);
  uint16_t* seg = reinterpret_cast<uint16_t*>(sm + S::seg);
  uint16_t* rnk = reinterpret_cast<uint16_t*>(sm + S::rnk);
  uint32_t* sl = reinterpret_cast<uint32_t*>(sm + S::sl);
  uint16_t* sq = reinterpret_cast<uint16_t*>(sm + S::sq);
  uint8_t* sop = sm + S::ops;
  __shared__ uint32_t s_bad, s_fail;
  __shared__ unsigned long long s_tally[MAXD], s_nins;
  const int tid = threadIdx.x, d = a.d, n = a.n, N = d * n, z = a.z;
  blk_stamp(0);
  if (tid == 0) s_bad = NONE32, s_fail = NONE32, s_nins = 0;
  if (tid < MAXD) s_tally[tid] = 0;
  // ---- 0. op codes: any code but 0 / 1 rejects the batch before anything is applied
  for (int t = tid; t < n; t += BLK_T) {
    const uint8_t o = a.ops[t];
    sop[t] = o;
    if (o > 1) atomicMin(&s_bad, (uint32_t)t);
  }
  __syncthreads();
  if (s_bad != NONE32) {
    if (tid == 0) {
      a.result[0] = SFK_BAD_OPCODE;
      a.result[1] = (int64_t)s_bad;
      a.result[2] = 0;
    }
    return;
  }
  // ---- 1. (cell, value) pairs, pair e = t * d + i, sorted by cell (stable:
  // a cell's pairs stay in stream order)
  uint32_t kk[IPT], vv[IPT];
#pragma unroll
  for (int q = 0; q < IPT; ++q) {
    const int e = tid * IPT + q;
    kk[q] = U32MAX;
    vv[q] = 0;
    if (e < N) {
      const int t = e / d, i = e - t * d;
      const uint64_t key = load_key(a.keys, t);
      kk[q] = (uint32_t)i * (uint32_t)a.w + (uint32_t)bucket(key, a.s_seeds.s[i], a.wm);
      vv[q] = ((uint32_t)t << 8) | ((uint32_t)i << 4) | ((uint32_t)sop[t] << 3) | (uint32_t)bucket(key, a.f_seeds.s[i], a.zm);
    }
  }
  BlkSort<IPT>(*reinterpret_cast<typename BlkSort<IPT>::TempStorage*>(sm + S::tmp)).Sort(kk, vv, 0, a.kbits + 1);
#pragma unroll
  for (int q = 0; q < IPT; ++q) sk[tid * IPT + q] = kk[q], sv[tid * IPT + q] = vv[q];  // padding last
  __syncthreads();
  blk_stamp(1);
  // ---- 2. fat counts: a segmented scan over the sorted pairs (thread tid
  // holds pairs tid * 8 .. tid * 8 + 7) of each cell's per-slot counts. A
  // cell's first pair carries the bucket's counts before the batch, so every
  // prefix is absolute; a cell's last pair writes the bucket back. Buckets are
  // read before the scan's barriers and written after them, except the
  // thread's own cells, read (again) before the thread writes them.
  BStateOp<Z> bop;
  const int e0 = tid * IPT;
  BState<Z> agg;
  agg.flag = 0;
  agg.head = 0;
#pragma unroll
  for (int k = 0; k < Z; ++k) agg.v[k] = 0;
  int lasthead = -1;     // the thread's last cell start: its cell may end in a later thread
  uint32_t linit[Z];     //   and its bucket, read before the scan
#pragma unroll
  for (int k = 0; k < Z; ++k) linit[k] = 0;
#pragma unroll
  for (int q = 0; q < IPT; ++q) {
    const int e = e0 + q;
    if (e >= N) break;
    BState<Z> el;
    el.flag = e == 0 || (q ? kk[q - 1] : sk[e - 1]) != kk[q];
    el.head = (uint32_t)e;
    const uint32_t dl = ((vv[q] >> 3) & 1u) ? U32MAX : 1u;
#pragma unroll
    for (int k = 0; k < Z; ++k) el.v[k] = (k == (int)(vv[q] & 7u)) ? dl : 0u;
    if (el.flag) {
      const uint32_t* fb = a.fat + (size_t)kk[q] * z;
#pragma unroll
      for (int k = 0; k < Z; ++k) {
        linit[k] = k < z ? fb[k] : 0u;
        el.v[k] += linit[k];
      }
      lasthead = q;
    }
    agg = q == 0 ? el : bop(agg, el);
  }
  BState<Z> run;
  __syncthreads();  // the sort's temp storage is reused by the scan
  cub::BlockScan<BState<Z>, BLK_T>(*reinterpret_cast<typename cub::BlockScan<BState<Z>, BLK_T>::TempStorage*>(sm + S::tmp))
      .ExclusiveScan(agg, run, bop);  // (thread 0's prefix is undefined and unused)
  __syncthreads();  // the scan's temp storage becomes obs
  blk_stamp(2);
  uint32_t fail = NONE32;
  {  // the slim value of every cell that starts here (independent loads first)
    uint32_t sv0[IPT];
#pragma unroll
    for (int q = 0; q < IPT; ++q) {
      const int e = e0 + q;
      const bool head = e < N && (e == 0 || (q ? kk[q - 1] : sk[e - 1]) != kk[q]);
      sv0[q] = head ? a.slim[kk[q]] : 0u;
    }
#pragma unroll
    for (int q = 0; q < IPT; ++q) {
      const int e = e0 + q;
      if (e < N && (e == 0 || (q ? kk[q - 1] : sk[e - 1]) != kk[q])) sl[e] = sv0[q], sq[e] = 0;
    }
  }
#pragma unroll
  for (int q = 0; q < IPT; ++q) {
    const int e = e0 + q;
    if (e >= N) break;
    const uint32_t c = kk[q], v = vv[q];
    const bool head = e == 0 || (q ? kk[q - 1] : sk[e - 1]) != c;
    const uint32_t k = v & 7u, op = (v >> 3) & 1u, row = (v >> 4) & 15u, t = v >> 8;
    BState<Z> el;
    el.flag = head;
    el.head = (uint32_t)e;
#pragma unroll
    for (int kq = 0; kq < Z; ++kq) el.v[kq] = (kq == (int)k) ? (op ? U32MAX : 1u) : 0u;
    if (head) {
      // a cell that starts and ends in this thread: its bucket is unwritten
      // until this thread writes it below
      const uint32_t* fb = a.fat + (size_t)c * z;
#pragma unroll
      for (int kq = 0; kq < Z; ++kq) el.v[kq] += q == lasthead ? linit[kq] : (kq < z ? fb[kq] : 0u);
    }
    run = (q == 0 && tid == 0) ? el : bop(run, el);
    uint32_t own_after = 0;
#pragma unroll
    for (int kq = 0; kq < Z; ++kq)
      if (kq == (int)k) own_after = run.v[kq];
    uint32_t ob;
    if (op == 0) {
      if (own_after == 0u) fail = min(fail, t);  // the count before was U32MAX
      ob = own_after;
    } else {
      if (own_after == U32MAX) fail = min(fail, t);  // the count before was 0
      if (a.variant == 1) {
        ob = 0;
#pragma unroll
        for (int kq = 0; kq < Z; ++kq) ob = max(ob, run.v[kq]);
      } else {
        unsigned long long sum = 0;
#pragma unroll
        for (int kq = 0; kq < Z; ++kq) sum += run.v[kq];
        ob = (uint32_t)min(sum, (unsigned long long)U32MAX);
      }
    }
    const int pr = (int)t * d + (int)row;
    obs[pr] = ob;
    seg[pr] = (uint16_t)run.head;
    rnk[pr] = (uint16_t)(e - (int)run.head);
    if (e + 1 == N || (q + 1 < IPT ? kk[q + 1] : sk[e + 1]) != c) {  // the cell's last pair
      uint32_t* fb = a.fat + (size_t)c * z;
#pragma unroll
      for (int kq = 0; kq < Z; ++kq)
        if (kq < z) fb[kq] = run.v[kq];
    }
  }
  if (fail != NONE32) atomicMin(&s_fail, fail);
  __syncthreads();
  blk_stamp(3);
  const uint32_t tf = s_fail;
  const int nv = (int)min((uint32_t)n, tf);  // ops applied: those before the first failing one
  // ---- 3. dataflow replay of the slim updates. Warp wp applies, in stream
  // order, the ops whose row-0 cell it owns (lane i on row i). An op first
  // waits until each of its cells has applied every earlier op on it; a cell
  // the warp itself touched last (rank = its last rank + 1) is already
  // current in the lane's register. The next op's records are loaded while
  // the current one is applied.
  {
    const int wp = tid >> 5, lane = tid & 31;
    uint32_t tally = 0, nins = 0;
    uint32_t csg = U32MAX, crk = 0, cs = 0;  // the lane's cached cell, its last rank there and its value
    int t0 = -32;
    unsigned mine = 0;
    // the warp's next op (stream order), or -1
    auto next_op = [&]() -> int {
      while (!mine) {
        t0 += 32;
        if (t0 >= nv) return -1;
        // op t belongs to the warp of its row-0 cell (a key's ops stay in one warp)
        mine = __ballot_sync(0xFFFFFFFFu, t0 + lane < nv && (seg[(t0 + lane) * d] & 31u) == (uint32_t)wp);
      }
      const int t = t0 + __ffs(mine) - 1;
      mine &= mine - 1u;
      return t;
    };
    uint32_t op = 0, sg = U32MAX, rk = 0, b = U32MAX;
    auto load_op = [&](int t) {
      op = sop[t];
      uint32_t ob = U32MAX;
      sg = U32MAX;
      rk = 0;
      if (lane < d) {
        sg = seg[t * d + lane];
        rk = rnk[t * d + lane];
        ob = obs[t * d + lane];
      }
      // an insert needs b_min = the min over the rows; a delete, the row's own cap
      b = op == 0 ? __reduce_min_sync(0xFFFFFFFFu, ob) : ob;
    };
    int t = next_op();
    if (t >= 0) load_op(t);
    while (t >= 0) {
      const uint32_t c_op = op, c_sg = sg, c_rk = rk, c_b = b;
      t = next_op();
      if (t >= 0) load_op(t);  // in flight while this op is applied
      const bool hit = lane >= d || (c_sg == csg && c_rk == crk + 1u);
      if (!__all_sync(0xFFFFFFFFu, hit)) {
        while (!__all_sync(0xFFFFFFFFu, hit || ld_acq16(sq + c_sg) == c_rk)) {
        }
        if (!hit) cs = sl[c_sg];
      }
      uint32_t s1 = cs;
      if (c_op == 0) {
        const uint32_t m = __reduce_min_sync(0xFFFFFFFFu, lane < d ? cs : U32MAX);
        if (m < c_b && lane < d && cs == m) s1 = cs + 1u, ++tally;
        ++nins;
      } else if (lane < d) {
        if (a.variant == 1) s1 = min(cs, c_b);
        else if (cs > c_b) s1 = cs - 1u;
      }
      if (lane < d) {
        if (s1 != cs) sl[c_sg] = s1;
        st_rel16(sq + c_sg, c_rk + 1u);
      }
      cs = s1;
      csg = c_sg;
      crk = c_rk;
    }
    if (lane < d && tally) atomicAdd(&s_tally[lane], (unsigned long long)tally);
    if (lane == 0 && nins) atomicAdd(&s_nins, (unsigned long long)nins);
  }
  __syncthreads();
  blk_stamp(4);
  // ---- 4. write back: slim cells; on a failing op, take its and the later
  // ops' fat deltas back (phase 2 counted every op; mod 2^32, exact)
  for (int e = tid; e < N; e += BLK_T) {
    const uint32_t c = sk[e];
    if (e > 0 && sk[e - 1] == c) continue;
    a.slim[c] = sl[e];
  }
  if (tf != NONE32) {
    for (int pr = (int)tf * d + tid; pr < N; pr += BLK_T) {
      const int t = pr / d, row = pr - t * d;
      const uint32_t c = sk[seg[pr]];
      const uint32_t k = (uint32_t)bucket(load_key(a.keys, t), a.f_seeds.s[row], a.zm);
      atomicAdd(a.fat + (size_t)c * z + k, sop[t] == 0 ? U32MAX : 1u);
    }
  }
  if (tid < d) a.inc[tid] += (int64_t)s_tally[tid];
  if (tid == 0) {
    if (tf == NONE32) {
      a.result[0] = SFK_OK;
      a.result[1] = -1;
    } else {
      a.result[0] = sop[tf] == 0 ? SFK_SATURATED : SFK_PHANTOM;
      a.result[1] = (int64_t)tf;
    }
    a.result[2] = (int64_t)s_nins;
  }
  blk_stamp(5);
}

int blk_profile(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, g_blk_prof, sizeof(unsigned long long) * 6);
}

// whether a batch's shape fits the block engine (the device's opt-in shared
// memory is checked at launch)
bool blk_fits(int d, int64_t w, int64_t z, int64_t n) {
  return d >= 1 && d <= MAXD && z >= 1 && z <= BLK_ZMAX && n >= 1 && (int64_t)d * n <= BLK_N &&
         (uint64_t)d * (uint64_t)w < (1ull << 31);
}

// the block engine for an SFF (variant 1) / SF4 (variant 0) batch, or -1 if
// the batch does not fit it
int launch_blk_bucket(int variant, uint32_t* slim, uint32_t* fat, const uint64_t* s_seeds, const uint64_t* f_seeds,
                      int d, int64_t w, int64_t z, const uint8_t* ops, KeySrc ks, int64_t n, int64_t* inc,
                      int64_t* result, cudaStream_t st) {
  if (!blk_fits(d, w, z, n)) return -1;  // (cell ids stay below the sort's padding key)
  BlkArgs a{};
  a.slim = slim;
  a.fat = fat;
  for (int i = 0; i < d; ++i) a.s_seeds.s[i] = s_seeds[i], a.f_seeds.s[i] = f_seeds[i];
  a.d = d;
  a.z = (int)z;
  a.n = (int)n;
  a.variant = variant;
  a.w = w;
  a.wm = make_mod((uint64_t)w);
  a.zm = make_mod((uint64_t)z);
  int kb = 1;
  while (kb < 32 && ((uint64_t)1 << kb) < (uint64_t)d * (uint64_t)w) ++kb;
  a.kbits = kb;
  a.ops = ops;
  a.keys = ks;
  a.inc = inc;
  a.result = result;
  int Z = 1;
  while (Z < z) Z <<= 1;
  auto launch = [&](auto kern, size_t smem) -> int {
    // the opt-in belongs to the current device's context: set it per call
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
      cudaGetLastError();
      return -1;
    }
    note_launch();
    kern<<<1, BLK_T, smem, st>>>(a);
    return check_launch("blk_bucket");
  };
  const int64_t N = (int64_t)d * n;
  const int ipt = N <= 2 * BLK_T ? 2 : N <= 4 * BLK_T ? 4 : 8;
#define SFK_BLK_CASE(ZZ)                                                          \
  case ZZ:                                                                        \
    return ipt == 2 ? launch(blk_bucket_k<ZZ, 2>, BlkSmem<ZZ>::total)             \
         : ipt == 4 ? launch(blk_bucket_k<ZZ, 4>, BlkSmem<ZZ>::total)             \
                    : launch(blk_bucket_k<ZZ, 8>, BlkSmem<ZZ>::total);
  switch (Z) {
    SFK_BLK_CASE(1)
    SFK_BLK_CASE(2)
    SFK_BLK_CASE(4)
    default:
      SFK_BLK_CASE(8)
  }
#undef SFK_BLK_CASE
}

}  // namespace sfk
