// Device-side generator of the cfg-5 query stream and a
// launch counter. The generator is the counter-based construction of
// paper_1701_04148_b200.workloads.query_keys, evaluated on the GPU so a
// 1B-key batch never crosses PCIe; both sides produce identical keys.
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

// _kernels.interleave_deletions (_kernels.py:427-467): a sequential walk over
// the stream (each step depends on the live-item set), one device thread
__global__ void interleave_k(const int64_t* __restrict__ cand, const double* __restrict__ decide,
                             const double* __restrict__ pick, double p, int64_t n, int64_t* counts,
                             int64_t* poslist, int64_t* posindex, uint8_t* __restrict__ ops,
                             int64_t* __restrict__ ranks) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  int64_t npos = 0, cur = 0;
  for (int64_t t = 0; t < n; ++t) {
    if (decide[t] < p && npos > 0) {
      int64_t slot = (int64_t)(pick[t] * (double)npos);
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
      const int64_t r = cand[cur++];
      ops[t] = 0;
      ranks[t] = r;
      if (++counts[r] == 1) {
        poslist[npos] = r;
        posindex[r] = npos;
        ++npos;
      }
    }
  }
}

int launch_interleave(const int64_t* cand, const double* decide, const double* pick, double p, int64_t n, int64_t v,
                      uint8_t* ops, int64_t* ranks, void* ws, size_t ws_bytes, cudaStream_t st) {
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
