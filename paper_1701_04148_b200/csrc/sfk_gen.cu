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

}  // namespace sfk
