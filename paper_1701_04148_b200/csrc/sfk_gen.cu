// Device-side generator of the cfg-5 query stream and a
// launch counter. The generator is the counter-based construction of
// paper_1701_04148_b200.workloads.query_keys, evaluated on the GPU so a
// 1B-key batch never crosses PCIe; both sides produce identical keys.
#include <cub/cub.cuh>

#include "sfk_common.cuh"

namespace sfk {

__global__ void gen_query_keys_k(uint64_t seed, const uint32_t* __restrict__ present,
                                 const uint32_t* __restrict__ sorted_present, uint32_t v,
                                 const double* __restrict__ cdf, int64_t t0, int64_t n, uint32_t* __restrict__ out) {
  const uint64_t GOLDEN = 0x9E3779B97F4A7C15ull;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t t = (uint64_t)(t0 + q);
    const uint64_t h = mix64(seed + (t + 1) * GOLDEN);
    uint32_t key;
    if ((h & 1) == 0) {
      const double u = (double)(h >> 11) * (1.0 / 9007199254740992.0);
      int64_t r;
      if (cdf == nullptr) {
        r = (int64_t)(u * (double)v);
      } else {  // upper_bound: first i with cdf[i] > u (numpy searchsorted side="right")
        uint32_t lo = 0, hi = v;
        while (lo < hi) {
          uint32_t mid = (lo + hi) >> 1;
          if (cdf[mid] > u) hi = mid; else lo = mid + 1;
        }
        r = lo;
      }
      if (r > (int64_t)v - 1) r = v - 1;
      key = present[r];
    } else {
      for (uint64_t j = 1;; ++j) {
        const uint32_t cand = (uint32_t)(mix64(h ^ (j * GOLDEN)) & 0xFFFFFFFFull);
        uint32_t lo = 0, hi = v;
        while (lo < hi) {
          uint32_t mid = (lo + hi) >> 1;
          if (sorted_present[mid] < cand) lo = mid + 1; else hi = mid;
        }
        if (lo >= v || sorted_present[lo] != cand) { key = cand; break; }
      }
    }
    out[q] = key;
  }
}

int launch_gen_query_keys(uint64_t seed, const uint32_t* present, const uint32_t* sorted_present, uint32_t v,
                          const double* cdf, int64_t t0, int64_t n, uint32_t* out, cudaStream_t st) {
  if (n <= 0) return 0;
  { note_launch(); gen_query_keys_k<<<grid_for(n, 256, sm_count() * 16), 256, 0, st>>>(seed, present, sorted_present, v, cdf, t0, n,
                                                                      out); }
  return check_launch("gen_query_keys");
}

// ---------------------------------------------------------------- numpy PCG64 on the device
// The reference's synthetic streams (workloads.generate, workloads.py:106-131)
// draw from numpy's Generator(PCG64(seed)): a 128-bit LCG (multiplier
// 0x2360ED051FC65DA44385DF649FCCF645) stepped before each output, output
// XSL-RR (rotate (hi ^ lo) right by the top 6 state bits), random() =
// (out >> 11) 2^-53. The host hands over the seeded state / increment
// (numpy's SeedSequence); each thread jumps to its slice of the stream with
// the LCG's O(log k) advance, so any stretch is generated in parallel.
typedef unsigned __int128 u128;
__device__ __forceinline__ u128 pcg_mult() {
  return ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;
}
__device__ __forceinline__ uint64_t pcg_out(u128 s) {
  const uint64_t x = (uint64_t)(s >> 64) ^ (uint64_t)s;
  const unsigned rot = (unsigned)(s >> 122);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}
__device__ u128 pcg_advance(u128 s, u128 inc, uint64_t delta) {
  u128 cm = pcg_mult(), cp = inc, am = 1, ap = 0;
  while (delta) {
    if (delta & 1ull) {
      am *= cm;
      ap = ap * cm + cp;
    }
    cp = (cm + 1) * cp;
    cm *= cm;
    delta >>= 1;
  }
  return am * s + ap;
}

constexpr int PCG_CHUNK = 64;

// n doubles of the stream starting at draw `offset`; with a CDF, the
// reference's Zipf rank searchsorted(cdf, u, side="right") instead
__global__ void pcg_uniform_k(uint64_t sh, uint64_t sl, uint64_t ih, uint64_t il, int64_t offset, int64_t n,
                              const double* __restrict__ cdf, int64_t v, int64_t* __restrict__ ranks,
                              double* __restrict__ uout) {
  const u128 s0 = ((u128)sh << 64) | sl, inc = ((u128)ih << 64) | il;
  const int64_t nchunks = (n + PCG_CHUNK - 1) / PCG_CHUNK;
  for (int64_t ch = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; ch < nchunks;
       ch += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = ch * PCG_CHUNK, b = min(n, a + PCG_CHUNK);
    u128 s = pcg_advance(s0, inc, (uint64_t)(offset + a));
    const u128 M = pcg_mult();
    for (int64_t i = a; i < b; ++i) {
      s = s * M + inc;
      const double u = (double)(pcg_out(s) >> 11) * (1.0 / 9007199254740992.0);
      if (cdf) {
        int64_t lo = 0, hi = v;
        while (lo < hi) {
          const int64_t mid = (lo + hi) >> 1;
          if (cdf[mid] > u) hi = mid; else lo = mid + 1;
        }
        ranks[i] = lo;
      } else {
        uout[i] = u;
      }
    }
  }
}

int launch_pcg_uniform(uint64_t sh, uint64_t sl, uint64_t ih, uint64_t il, int64_t offset, int64_t n,
                       const double* cdf, int64_t v, int64_t* ranks, double* uout, cudaStream_t st) {
  if (n <= 0) return 0;
  const int64_t nchunks = (n + PCG_CHUNK - 1) / PCG_CHUNK;
  { note_launch(); pcg_uniform_k<<<grid_for(nchunks, 128, sm_count() * 16), 128, 0, st>>>(sh, sl, ih, il, offset, n, cdf, v, ranks, uout); }
  return check_launch("pcg_uniform");
}

// numpy's Generator.integers(0, v) for int64 (v <= 2^32): 32-bit draws taken
// from each 64-bit output low half first, Lemire's method with rejection
// (a draw u is accepted iff (u * v) mod 2^32 >= (2^32 - v) mod v; the value
// is (u * v) >> 32). Acceptance depends on the draw alone, so sample i is the
// i-th accepted 32-bit position: flag every position in parallel, compact.
__global__ void pcg_bounded_flags_k(uint64_t sh, uint64_t sl, uint64_t ih, uint64_t il, int64_t offset64, int64_t k32,
                                    uint32_t v, uint32_t thr, uint8_t* __restrict__ flag, int64_t* __restrict__ val) {
  const u128 s0 = ((u128)sh << 64) | sl, inc = ((u128)ih << 64) | il;
  const int64_t n64 = (k32 + 1) / 2;
  const int64_t nchunks = (n64 + PCG_CHUNK - 1) / PCG_CHUNK;
  for (int64_t ch = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; ch < nchunks;
       ch += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = ch * PCG_CHUNK, b = min(n64, a + PCG_CHUNK);
    u128 st = pcg_advance(s0, inc, (uint64_t)(offset64 + a));
    const u128 M = pcg_mult();
    for (int64_t d = a; d < b; ++d) {
      st = st * M + inc;
      const uint64_t o = pcg_out(st);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t pos = 2 * d + h;
        if (pos >= k32) break;
        const uint32_t u = (uint32_t)(h ? (o >> 32) : o);
        if (v == 0) {  // v = 2^32: numpy returns the raw 32-bit draw
          flag[pos] = 1;
          val[pos] = (int64_t)u;
        } else {
          const uint64_t m = (uint64_t)u * (uint64_t)v;
          flag[pos] = (uint32_t)m >= thr ? 1 : 0;
          val[pos] = (int64_t)(m >> 32);
        }
      }
    }
  }
}

// 32-bit draws needed for n samples: the expected count n / (1 - thr / 2^32)
// plus 10 standard deviations (a shortfall is reported, never truncated)
int64_t pcg_bounded_window(int64_t n, int64_t v) {
  const double p = (double)((0x100000000ull - (uint64_t)v) % (uint64_t)v) / 4294967296.0;
  const double e = (double)n / (1.0 - p);
  return (int64_t)(e + 10.0 * sqrt(e + 1.0)) + 64;
}

static size_t bounded_tmp_bytes(int64_t k32) {
  size_t a = 0, b = 0;
  cub::DeviceSelect::Flagged(nullptr, a, (const int64_t*)nullptr, (const uint8_t*)nullptr, (int64_t*)nullptr,
                             (int64_t*)nullptr, k32);
  cub::DeviceSelect::Flagged(nullptr, b, cub::CountingInputIterator<int64_t>(0), (const uint8_t*)nullptr,
                             (int64_t*)nullptr, (int64_t*)nullptr, k32);
  return std::max(a, b);
}

size_t pcg_bounded_workspace_size(int64_t n, int64_t v) {
  const int64_t k32 = pcg_bounded_window(n, v);
  Carver cv(nullptr, ~size_t(0));
  cv.take<uint8_t>((size_t)k32);
  cv.take<int64_t>((size_t)k32);
  cv.take<int64_t>((size_t)k32);
  cv.take<int64_t>((size_t)k32);
  cv.take<int64_t>(2);
  cv.take<char>(bounded_tmp_bytes(k32));
  return cv.off + 256;
}

int launch_pcg_bounded(uint64_t sh, uint64_t sl, uint64_t ih, uint64_t il, int64_t offset64, int64_t n, int64_t v,
                       int64_t* out, int64_t* next_offset64, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (n <= 0) { *next_offset64 = offset64; return 0; }
  if (v == 1) {  // numpy's range 0: no draws, all zeros
    cudaMemsetAsync(out, 0, (size_t)n * 8, st);
    *next_offset64 = offset64;
    return check_launch("pcg_bounded");
  }
  const uint32_t vv = (uint32_t)v;  // 0 encodes v = 2^32 (raw draws)
  const uint32_t thr = (uint32_t)((0x100000000ull - (uint64_t)v) % (uint64_t)v);
  const int64_t k32 = pcg_bounded_window(n, v);
  Carver cv(ws, ws_bytes);
  uint8_t* flag = cv.take<uint8_t>((size_t)k32);
  int64_t* val = cv.take<int64_t>((size_t)k32);
  int64_t* acc = cv.take<int64_t>((size_t)k32);
  int64_t* pos = cv.take<int64_t>((size_t)k32);
  int64_t* sel = cv.take<int64_t>(2);
  const size_t tb = bounded_tmp_bytes(k32);
  void* tmp = cv.take<char>(tb);
  if (!cv.ok || ws == nullptr) {
    set_error("bounded draws: workspace too small (need %zu bytes)", cv.off + 256);
    return 1;
  }
  const int64_t n64 = (k32 + 1) / 2, nchunks = (n64 + PCG_CHUNK - 1) / PCG_CHUNK;
  { note_launch(); pcg_bounded_flags_k<<<grid_for(nchunks, 128, sm_count() * 16), 128, 0, st>>>(sh, sl, ih, il, offset64, k32, vv, thr, flag, val); }
  size_t b1 = tb;
  if (cub::DeviceSelect::Flagged(tmp, b1, val, flag, acc, sel, k32, st) != cudaSuccess) return 1;
  b1 = tb;
  if (cub::DeviceSelect::Flagged(tmp, b1, cub::CountingInputIterator<int64_t>(0), flag, pos, sel + 1, k32, st) !=
      cudaSuccess)
    return 1;
  int64_t h[2];
  cudaMemcpyAsync(h, sel, 16, cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) { set_error("bounded draws: sync failed"); return 1; }
  if (h[0] < n) {
    set_error("bounded draws: %lld accepted of %lld needed in the window", (long long)h[0], (long long)n);
    return 1;
  }
  cudaMemcpyAsync(out, acc, (size_t)n * 8, cudaMemcpyDeviceToDevice, st);
  int64_t last = 0;
  cudaMemcpyAsync(&last, pos + (n - 1), 8, cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) { set_error("bounded draws: sync failed"); return 1; }
  *next_offset64 = offset64 + (last + 2) / 2;  // 32-bit draws used: last + 1; a half-used 64-bit draw is dropped
  return check_launch("pcg_bounded");
}

// _kernels.interleave_deletions (_kernels.py:427-467): a sequential walk over
// the stream (each step depends on the live-item set), one device thread
__global__ void interleave_k(const int64_t* __restrict__ cand, const double* __restrict__ decide,
                             const double* __restrict__ pick, double p, int64_t n, int64_t* counts,
                             int64_t* poslist, int64_t* posindex, uint8_t* __restrict__ ops,
                             int64_t* __restrict__ ranks) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  int64_t npos = 0, cur = 0;
  constexpr int B = 8;  // decide / pick / candidate draws loaded B at a time
  for (int64_t t0 = 0; t0 < n; t0 += B) {
    double dd[B], pp[B];
    int64_t cc[B];
#pragma unroll
    for (int q = 0; q < B; ++q) {
      dd[q] = t0 + q < n ? __ldg(decide + t0 + q) : 1.0;
      pp[q] = t0 + q < n ? __ldg(pick + t0 + q) : 0.0;
      cc[q] = cur + q < n ? __ldg(cand + cur + q) : 0;
    }
    int used = 0;
#pragma unroll
    for (int q = 0; q < B; ++q) {
      const int64_t t = t0 + q;
      if (t >= n) break;
      if (dd[q] < p && npos > 0) {
        int64_t slot = (int64_t)(pp[q] * (double)npos);
        if (slot >= npos) slot = npos - 1;
        const int64_t r = poslist[slot];
        ops[t] = 1;
        ranks[t] = r;
        if (--counts[r] == 0) {
          const int64_t last = poslist[npos - 1];
          poslist[slot] = last;
          posindex[last] = slot;
          posindex[r] = -1;
          --npos;
        }
      } else {
        int64_t r = cc[0];
#pragma unroll
        for (int u = 1; u < B; ++u)
          if (u == used) r = cc[u];
        ++used;
        ops[t] = 0;
        ranks[t] = r;
        if (++counts[r] == 1) {
          poslist[npos] = r;
          posindex[r] = npos;
          ++npos;
        }
      }
    }
    cur += used;
  }
}

// the same walk with the live-item tables in shared memory (v small enough):
// each step's table accesses cost shared-memory latency instead of L2's
__global__ void __launch_bounds__(256) interleave_smem_k(const int64_t* __restrict__ cand,
                                                         const double* __restrict__ decide,
                                                         const double* __restrict__ pick, double p, int64_t n,
                                                         int32_t v, uint8_t* __restrict__ ops,
                                                         int64_t* __restrict__ ranks) {
  extern __shared__ int32_t tab[];
  int32_t* counts = tab;
  int32_t* poslist = tab + v;
  int32_t* posindex = tab + 2 * v;
  for (int32_t r = threadIdx.x; r < v; r += blockDim.x) counts[r] = 0;
  __syncthreads();
  if (threadIdx.x != 0) return;
  int32_t npos = 0;
  int64_t cur = 0;
  constexpr int B = 8;  // decide / pick / candidate draws loaded B at a time
  for (int64_t t0 = 0; t0 < n; t0 += B) {
    double dd[B], pp[B];
    int64_t cc[B];
#pragma unroll
    for (int q = 0; q < B; ++q) {
      dd[q] = t0 + q < n ? __ldg(decide + t0 + q) : 1.0;
      pp[q] = t0 + q < n ? __ldg(pick + t0 + q) : 0.0;
      cc[q] = cur + q < n ? __ldg(cand + cur + q) : 0;
    }
    int used = 0;
#pragma unroll
    for (int q = 0; q < B; ++q) {
      const int64_t t = t0 + q;
      if (t >= n) break;
      if (dd[q] < p && npos > 0) {
        int64_t slot = (int64_t)(pp[q] * (double)npos);
        if (slot >= npos) slot = npos - 1;
        const int32_t r = poslist[slot];
        ops[t] = 1;
        ranks[t] = r;
        if (--counts[r] == 0) {
          const int32_t last = poslist[npos - 1];
          poslist[slot] = last;
          posindex[last] = (int32_t)slot;
          posindex[r] = -1;
          --npos;
        }
      } else {
        // the next candidate: one of the B prefetched (inserts consume them in order)
        int64_t rr = cc[0];
#pragma unroll
        for (int u = 1; u < B; ++u)
          if (u == used) rr = cc[u];
        ++used;
        const int32_t r = (int32_t)rr;
        ops[t] = 0;
        ranks[t] = r;
        if (++counts[r] == 1) {
          poslist[npos] = r;
          posindex[r] = npos;
          ++npos;
        }
      }
    }
    cur += used;
  }
}

int launch_interleave(const int64_t* cand, const double* decide, const double* pick, double p, int64_t n, int64_t v,
                      uint8_t* ops, int64_t* ranks, void* ws, size_t ws_bytes, cudaStream_t st) {
  {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    const size_t smem = (size_t)v * 3 * 4;
    if (v < (int64_t)1 << 30 && smem + 1024 <= (size_t)optin) {
      if (smem > 48 * 1024 &&
          cudaFuncSetAttribute(interleave_smem_k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
              cudaSuccess) {
        cudaGetLastError();
      } else {
        if (n > 0) { note_launch(); interleave_smem_k<<<1, 256, smem, st>>>(cand, decide, pick, p, n, (int32_t)v, ops, ranks); }
        return check_launch("interleave_smem");
      }
    }
  }
  Carver cv(ws, ws_bytes);
  int64_t* counts = cv.take<int64_t>((size_t)v);
  int64_t* poslist = cv.take<int64_t>((size_t)v);
  int64_t* posindex = cv.take<int64_t>((size_t)v);
  if (!cv.ok || ws == nullptr) {
    set_error("interleave workspace too small: need %zu bytes", cv.off);
    return 1;
  }
  cudaMemsetAsync(counts, 0, (size_t)v * 8, st);
  if (n > 0) { note_launch(); interleave_k<<<1, 1, 0, st>>>(cand, decide, pick, p, n, counts, poslist, posindex, ops, ranks); }
  return check_launch("interleave");
}

}  // namespace sfk
