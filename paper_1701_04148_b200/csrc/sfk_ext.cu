// The signed-median Count sketch and the log-counter (CML) sketch on the GPU
// (sfsketch.baselines.CountSketch / CmlSketch, baselines.py:90-128,182-238).
//
// Count updates commute (signed +-1 per row), so a batch that cannot reach a
// saturated counter (checked on the device from the counter extremes and the
// batch length) is one pass of warp-aggregated atomics; any other batch goes
// to the exact sequential device engine. Count queries: 2d hashes, d
// gathers, an in-register sort and the reference's median rule.
// CML updates are ordered (gated min-raise); they run in the ordered slim
// engine (sfk_sf.cu, kind 7). CML queries: the min exponent over the d rows,
// optionally decoded through a caller-provided value table.
#include "sfk_common.cuh"

namespace sfk {

constexpr uint64_t SIGN_SALT = 0xA5A5A5A5A5A5A5A5ull;  // _kernels.py:37

// per-row sign (_kernels.py:129-130): +1 when bit 0 of finalize64(key ^ seed ^ salt) is 0
__device__ __forceinline__ int count_sign(uint64_t key, uint64_t seed) {
  return (mix64(key ^ seed ^ SIGN_SALT) & 1ull) ? -1 : 1;
}

// Lanes of a warp that hit the same cell merge their signed deltas
// (__match_any_sync + __reduce_add_sync); the group leader issues one atomic.
template <int D>
__global__ void __launch_bounds__(256) count_atomic_k(int32_t* __restrict__ counters, Seeds<D> seeds, Mod wm,
                                                      uint32_t w, const uint8_t* __restrict__ ops, KeySrc keys,
                                                      int64_t n) {
  const int lane = threadIdx.x & 31;
  const int64_t warp_id = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = warp_id * 32; base < n; base += nwarps * 32) {
    const int64_t t = base + lane;
    const bool active = t < n;
    const unsigned amask = __ballot_sync(0xffffffffu, active);
    if (!active) continue;
    const uint64_t key = load_key(keys, t);
    const int flip = ops[t] ? -1 : 1;
#pragma unroll
    for (int i = 0; i < D; ++i) {
      const uint32_t cell = (uint32_t)i * w + (uint32_t)bucket(key, seeds.s[i], wm);
      const int dl = count_sign(key, seeds.s[i]) * flip;
      const unsigned g = __match_any_sync(amask, cell);
      const int net = __reduce_add_sync(g, dl);
      if (lane == __ffs(g) - 1 && net) atomicAdd(counters + cell, net);
    }
  }
}

// count_query (_kernels.py:149-179): median of the sign-corrected reads; even
// d: mean of the central pair rounded half away from zero; clamped at 0.
__device__ __forceinline__ int64_t median_rule(const int64_t* buf, int d) {
  int64_t med;
  if (d & 1) {
    med = buf[d / 2];
  } else {
    const int64_t pair = buf[d / 2 - 1] + buf[d / 2];
    if ((pair & 1) == 0) med = pair / 2;
    else if (pair > 0) med = (pair + 1) / 2;
    else med = (pair - 1) / 2;
  }
  return med < 0 ? 0 : med;
}

template <int D>
__global__ void __launch_bounds__(256) count_query_k(const int32_t* __restrict__ c, Seeds<D> seeds, Mod wm, uint32_t w,
                                                     KeySrc keys, int64_t n, int64_t* __restrict__ out) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = load_key(keys, t);
    int64_t buf[D];
#pragma unroll
    for (int i = 0; i < D; ++i) {
      const int64_t v = __ldg(c + (size_t)i * w + bucket(key, seeds.s[i], wm));
      buf[i] = count_sign(key, seeds.s[i]) > 0 ? v : -v;
    }
    // sorting network by odd-even transposition: static indices, registers only
#pragma unroll
    for (int r = 0; r < D; ++r) {
#pragma unroll
      for (int i = r & 1; i + 1 < D; i += 2) {
        const int64_t a = buf[i], b = buf[i + 1];
        buf[i] = min(a, b);
        buf[i + 1] = max(a, b);
      }
    }
    out[t] = median_rule(buf, D);
  }
}

// d > 8: one thread per key, local-memory sort
__global__ void __launch_bounds__(128) count_query_dyn_k(const int32_t* __restrict__ c, Seeds<MAXSEEDS> seeds, int d,
                                                         Mod wm, uint32_t w, KeySrc keys, int64_t n,
                                                         int64_t* __restrict__ out) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = load_key(keys, t);
    int64_t buf[MAXSEEDS];
    for (int i = 0; i < d; ++i) {
      const int64_t v = c[(size_t)i * w + bucket(key, seeds.s[i], wm)];
      buf[i] = count_sign(key, seeds.s[i]) > 0 ? v : -v;
    }
    for (int a = 1; a < d; ++a) {
      const int64_t x = buf[a];
      int b = a - 1;
      while (b >= 0 && buf[b] > x) { buf[b + 1] = buf[b]; --b; }
      buf[b + 1] = x;
    }
    out[t] = median_rule(buf, d);
  }
}

// cml_min_exp (_kernels.py:214-226), decoded through vtab when given
template <int D>
__global__ void __launch_bounds__(256) cml_query_k(const uint16_t* __restrict__ e, Seeds<D> seeds, Mod wm, uint32_t w,
                                                   KeySrc keys, int64_t n, const int64_t* __restrict__ vtab,
                                                   int64_t* __restrict__ out) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = load_key(keys, t);
    uint32_t best = 0xFFFFu;
#pragma unroll
    for (int i = 0; i < D; ++i) best = min(best, (uint32_t)__ldg(e + (size_t)i * w + bucket(key, seeds.s[i], wm)));
    out[t] = vtab ? __ldg(vtab + best) : (int64_t)best;
  }
}

__global__ void __launch_bounds__(128) cml_query_dyn_k(const uint16_t* __restrict__ e, Seeds<MAXSEEDS> seeds, int d,
                                                       Mod wm, uint32_t w, KeySrc keys, int64_t n,
                                                       const int64_t* __restrict__ vtab, int64_t* __restrict__ out) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = load_key(keys, t);
    uint32_t best = 0xFFFFu;
    for (int i = 0; i < d; ++i) best = min(best, (uint32_t)e[(size_t)i * w + bucket(key, seeds.s[i], wm)]);
    out[t] = vtab ? vtab[best] : (int64_t)best;
  }
}

int sm_count();

// Preconditions of the gated engine kinds, checked on the device. The
// ordered engine caps each op at a u32 (the oracle's true count, the CML
// exponent bound), which is exact as long as no op can meet a saturated
// minimum:
// * oracle-assisted: the reference compares against np.uint64(true_count),
//   so a negative or >= 2^32 count is a cap above every u32 minimum; capping
//   it at 2^32 - 1 is exact unless a slim cell can reach 2^32 - 1 within the
//   batch (max cell + n < 2^32 - 1 rules that out);
// * CML: a non-increasing gate table (so "uf < gate[c]" equals "c < first c
//   with gate[c] <= uf"), and the 0xFFFF exponent out of reach: gate[65535]
//   == 0, or max exponent + n < 0xFFFF.
// flag[0]: gate not monotone; [1]: gate[65535] != 0; [2]: max exponent;
// [3]: a count above 2^32 - 1 as u64; [4]: max slim cell.
__global__ void gated_precheck_k(const int64_t* __restrict__ tc, int64_t n, const double* __restrict__ gate,
                                 const uint16_t* __restrict__ exps, const uint32_t* __restrict__ slim, int64_t cells,
                                 unsigned* __restrict__ flag) {
  unsigned bad = 0, big = 0, mx = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tc)
    for (int64_t t = tid; t < n; t += stride) big |= (uint64_t)tc[t] > 0xFFFFFFFFull;
  if (gate) {
    for (int64_t i = tid; i + 1 < 65536; i += stride) bad |= gate[i + 1] > gate[i];
    if (tid == 0 && gate[65535] != 0.0) flag[1] = 1u;
  }
  if (exps)
    for (int64_t c = tid; c < cells; c += stride) mx = max(mx, (unsigned)exps[c]);
  if (slim)
    for (int64_t c = tid; c < cells; c += stride) mx = max(mx, slim[c]);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1u);
  if (__any_sync(0xffffffffu, big) && (threadIdx.x & 31) == 0) atomicOr(flag + 3, 1u);
  for (int off = 16; off > 0; off >>= 1) mx = max(mx, __shfl_down_sync(0xffffffffu, mx, off));
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(flag + (exps ? 2 : 4), mx);
}

static int64_t ext_grid(int64_t n, int threads) {
  const int64_t cap = (int64_t)sm_count() * 16;
  int64_t g = (n + threads - 1) / threads;
  return g < 1 ? 1 : (g > cap ? cap : g);
}

template <int D>
static int count_fast_d(int32_t* counters, const uint64_t* seeds, int64_t w, const uint8_t* ops, KeySrc ks, int64_t n,
                        cudaStream_t st) {
  Seeds<D> sd;
  for (int i = 0; i < D; ++i) sd.s[i] = seeds[i];
  { note_launch(); count_atomic_k<D><<<ext_grid((n + 31) / 32 * 32, 256), 256, 0, st>>>(counters, sd, make_mod((uint64_t)w), (uint32_t)w, ops, ks, n); }
  return check_launch("count_atomic");
}

int count_fast(int32_t* counters, const uint64_t* seeds, int d, int64_t w, const uint8_t* ops, KeySrc ks, int64_t n,
               cudaStream_t st) {
  switch (d) {
    case 1: return count_fast_d<1>(counters, seeds, w, ops, ks, n, st);
    case 2: return count_fast_d<2>(counters, seeds, w, ops, ks, n, st);
    case 3: return count_fast_d<3>(counters, seeds, w, ops, ks, n, st);
    case 4: return count_fast_d<4>(counters, seeds, w, ops, ks, n, st);
    case 5: return count_fast_d<5>(counters, seeds, w, ops, ks, n, st);
    case 6: return count_fast_d<6>(counters, seeds, w, ops, ks, n, st);
    case 7: return count_fast_d<7>(counters, seeds, w, ops, ks, n, st);
    case 8: return count_fast_d<8>(counters, seeds, w, ops, ks, n, st);
  }
  set_error("count fast path: unsupported d=%d", d);
  return 1;
}

template <int D>
static int ext_query_d(int which, const void* table, const uint64_t* seeds, int64_t w, KeySrc ks, int64_t n,
                       const int64_t* vtab, int64_t* out, cudaStream_t st) {
  Seeds<D> sd;
  for (int i = 0; i < D; ++i) sd.s[i] = seeds[i];
  const Mod wm = make_mod((uint64_t)w);
  if (which == 0) {
    note_launch();
    count_query_k<D><<<ext_grid(n, 256), 256, 0, st>>>(static_cast<const int32_t*>(table), sd, wm, (uint32_t)w, ks, n, out);
  } else {
    note_launch();
    cml_query_k<D><<<ext_grid(n, 256), 256, 0, st>>>(static_cast<const uint16_t*>(table), sd, wm, (uint32_t)w, ks, n, vtab, out);
  }
  return check_launch(which == 0 ? "count_query" : "cml_query");
}

// which: 0 Count median, 1 CML min exponent (decoded through vtab if non-null)
int ext_query(int which, const void* table, const uint64_t* seeds, int d, int64_t w, KeySrc ks, int64_t n,
              const int64_t* vtab, int64_t* out, cudaStream_t st) {
  if (n <= 0) return 0;
  switch (d) {
    case 1: return ext_query_d<1>(which, table, seeds, w, ks, n, vtab, out, st);
    case 2: return ext_query_d<2>(which, table, seeds, w, ks, n, vtab, out, st);
    case 3: return ext_query_d<3>(which, table, seeds, w, ks, n, vtab, out, st);
    case 4: return ext_query_d<4>(which, table, seeds, w, ks, n, vtab, out, st);
    case 5: return ext_query_d<5>(which, table, seeds, w, ks, n, vtab, out, st);
    case 6: return ext_query_d<6>(which, table, seeds, w, ks, n, vtab, out, st);
    case 7: return ext_query_d<7>(which, table, seeds, w, ks, n, vtab, out, st);
    case 8: return ext_query_d<8>(which, table, seeds, w, ks, n, vtab, out, st);
  }
  Seeds<MAXSEEDS> sd;
  for (int i = 0; i < d; ++i) sd.s[i] = seeds[i];
  const Mod wm = make_mod((uint64_t)w);
  if (which == 0) {
    note_launch();
    count_query_dyn_k<<<ext_grid(n, 128), 128, 0, st>>>(static_cast<const int32_t*>(table), sd, d, wm, (uint32_t)w, ks, n, out);
  } else {
    note_launch();
    cml_query_dyn_k<<<ext_grid(n, 128), 128, 0, st>>>(static_cast<const uint16_t*>(table), sd, d, wm, (uint32_t)w, ks, n, vtab, out);
  }
  return check_launch(which == 0 ? "count_query" : "cml_query");
}

int gated_precheck(const int64_t* tc, int64_t n, const double* gate, const uint16_t* exps, const uint32_t* slim,
                   int64_t cells, void* ws, size_t ws_bytes, bool* ok, cudaStream_t st) {
  if (ws == nullptr || ws_bytes < 256) { set_error("workspace too small for the precheck"); return 1; }
  unsigned* flag = static_cast<unsigned*>(ws);
  cudaMemsetAsync(flag, 0, 32, st);
  int64_t work = 65536;
  if (tc && n > work) work = n;
  if (cells > work) work = cells;
  { note_launch(); gated_precheck_k<<<ext_grid(work, 256), 256, 0, st>>>(tc, tc ? n : 0, gate, exps, slim, cells, flag); }
  if (int r = check_launch("gated_precheck")) return r;
  unsigned h[8] = {1, 1, 0xFFFF, 1, 0xFFFFFFFFu, 0, 0, 0};
  cudaMemcpyAsync(h, flag, 32, cudaMemcpyDeviceToHost, st);
  const cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) { set_error("precheck: %s", cudaGetErrorString(e)); return (int)e; }
  *ok = h[0] == 0;
  if (gate && h[1] != 0) *ok = *ok && (int64_t)h[2] + n < 0xFFFF;
  if (tc && h[3] != 0) *ok = *ok && (int64_t)h[4] + n < (int64_t)0xFFFFFFFFll;
  return 0;
}

}  // namespace sfk
