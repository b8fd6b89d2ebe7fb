// Batched point query: fused key load + hash + d gathers + min
// (replaces _kernels.min_query, _kernels.py:229-241), plus mix_batch
// (_kernels.py:56-59) and key materialisation.
//
// Two kernels, chosen per call:
//   * L2 path: the counters stay in global memory (L2-resident for the
//     configs' 256 KiB - 1 MiB tables); every thread answers UNR keys per
//     iteration so UNR*d independent gathers are in flight.
//   * smem path: when d*w*4 fits the opt-in shared memory (cfg 4: 4x12800
//     u32 = 200 KiB) and the batch is large enough to amortise staging, one
//     persistent CTA per SM copies the whole table into shared memory once
//     and serves all its keys from there (measured ~7x the L2 gather rate).
#include "sfk_common.cuh"

namespace sfk {

template <int D, int UNR>
__global__ void __launch_bounds__(256) min_query_l2(const uint32_t* __restrict__ counters, Seeds<D> seeds,
                                                    Mod wm, int64_t w, KeySrc keys, int64_t n,
                                                    int64_t* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t base = t0; base < n; base += stride * UNR) {
    uint32_t v[UNR][D];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      int64_t t = base + (int64_t)u * stride;
      if (t < n) {
        uint64_t key = load_key(keys, t);
#pragma unroll
        for (int i = 0; i < D; ++i) {
          uint64_t j = bucket(key, seeds.s[i], wm);
          v[u][i] = __ldg(counters + (int64_t)i * w + (int64_t)j);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      int64_t t = base + (int64_t)u * stride;
      if (t < n) {
        uint32_t m = v[u][0];
#pragma unroll
        for (int i = 1; i < D; ++i) m = min(m, v[u][i]);
        out[t] = (int64_t)m;
      }
    }
  }
}

template <int D, int UNR>
__global__ void __launch_bounds__(1024) min_query_smem(const uint32_t* __restrict__ counters, Seeds<D> seeds,
                                                       Mod wm, int64_t w, KeySrc keys, int64_t n,
                                                       int64_t* __restrict__ out) {
  extern __shared__ uint4 smem_q[];
  uint32_t* tab = reinterpret_cast<uint32_t*>(smem_q);
  const int64_t words = (int64_t)D * w;
  // stage: 16-B vector loads when aligned, then the scalar tail
  const int64_t nvec = ((reinterpret_cast<uintptr_t>(counters) & 15) == 0) ? words / 4 : 0;
  const uint4* src4 = reinterpret_cast<const uint4*>(counters);
  for (int64_t k = threadIdx.x; k < nvec; k += blockDim.x) smem_q[k] = __ldg(src4 + k);
  for (int64_t k = nvec * 4 + threadIdx.x; k < words; k += blockDim.x) tab[k] = __ldg(counters + k);
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t base = t0; base < n; base += stride * UNR) {
    uint32_t m[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      int64_t t = base + (int64_t)u * stride;
      m[u] = U32MAX;
      if (t < n) {
        uint64_t key = load_key(keys, t);
#pragma unroll
        for (int i = 0; i < D; ++i) {
          uint32_t j = (uint32_t)bucket(key, seeds.s[i], wm);
          m[u] = min(m[u], tab[(uint32_t)(i * w) + j]);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      int64_t t = base + (int64_t)u * stride;
      if (t < n) out[t] = (int64_t)m[u];
    }
  }
}

// Any d up to MAXSEEDS: seeds passed by value.
__global__ void min_query_generic(const uint32_t* __restrict__ counters, Seeds<MAXSEEDS> seeds,
                                  int d, Mod wm, int64_t w, KeySrc keys, int64_t n, int64_t* __restrict__ out) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    uint64_t key = load_key(keys, t);
    uint32_t m = U32MAX;
    for (int i = 0; i < d; ++i) m = min(m, __ldg(counters + (int64_t)i * w + (int64_t)bucket(key, seeds.s[i], wm)));
    out[t] = (int64_t)m;
  }
}

__global__ void mix_batch_k(const uint64_t* __restrict__ keys, int64_t n, uint64_t* __restrict__ out) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    out[t] = mix64(keys[t]);
}

__global__ void load_keys_k(KeySrc keys, int64_t n, uint64_t* __restrict__ out) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    out[t] = load_key(keys, t);
}

template <int D>
static int launch_query_d(const uint32_t* counters, const uint64_t* seeds_host, int64_t w, KeySrc ks, int64_t n,
                          int64_t* out, cudaStream_t st) {
  Seeds<D> sd;
  for (int i = 0; i < D; ++i) sd.s[i] = seeds_host[i];
  Mod wm = make_mod((uint64_t)w);
  const int sms = sm_count();
  static int optin = -1;
  if (optin < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  }
  const size_t tab_bytes = (size_t)D * (size_t)w * 4;
  // staging costs tab_bytes per SM; worth it once the batch's own gathers
  // dwarf it (>= ~16 keys per staged counter word across the chip)
  if (tab_bytes <= (size_t)optin && (double)n * D >= 16.0 * (double)sms * (double)(D * w) / 4.0) {
    static bool attr_set = false;
    if (!attr_set) {
      cudaFuncSetAttribute(min_query_smem<D, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
      attr_set = true;
    }
    { note_launch(); min_query_smem<D, 4><<<sms, 1024, tab_bytes, st>>>(counters, sd, wm, w, ks, n, out); }
    return check_launch("min_query_smem");
  }
  int blocks = grid_for(n, 256 * 4, sms * 8);
  { note_launch(); min_query_l2<D, 4><<<blocks, 256, 0, st>>>(counters, sd, wm, w, ks, n, out); }
  return check_launch("min_query_l2");
}

int launch_min_query(const uint32_t* counters, const uint64_t* seeds_host, int d,
                     int64_t w, KeySrc ks, int64_t n, int64_t* out, cudaStream_t st) {
  if (n <= 0) return 0;
  switch (d) {
    case 1: return launch_query_d<1>(counters, seeds_host, w, ks, n, out, st);
    case 2: return launch_query_d<2>(counters, seeds_host, w, ks, n, out, st);
    case 3: return launch_query_d<3>(counters, seeds_host, w, ks, n, out, st);
    case 4: return launch_query_d<4>(counters, seeds_host, w, ks, n, out, st);
    case 5: return launch_query_d<5>(counters, seeds_host, w, ks, n, out, st);
    case 6: return launch_query_d<6>(counters, seeds_host, w, ks, n, out, st);
    case 7: return launch_query_d<7>(counters, seeds_host, w, ks, n, out, st);
    case 8: return launch_query_d<8>(counters, seeds_host, w, ks, n, out, st);
    default: {
      Mod wm = make_mod((uint64_t)w);
      Seeds<MAXSEEDS> sd;
      for (int i = 0; i < d && i < MAXSEEDS; ++i) sd.s[i] = seeds_host[i];
      { note_launch(); min_query_generic<<<grid_for(n, 256, sm_count() * 8), 256, 0, st>>>(counters, sd, d, wm, w, ks, n, out); }
      return check_launch("min_query_generic");
    }
  }
}

int launch_mix_batch(const uint64_t* keys, int64_t n, uint64_t* out, cudaStream_t st) {
  if (n <= 0) return 0;
  { note_launch(); mix_batch_k<<<grid_for(n, 256, sm_count() * 8), 256, 0, st>>>(keys, n, out); }
  return check_launch("mix_batch");
}

int launch_load_keys(KeySrc ks, int64_t n, uint64_t* out, cudaStream_t st) {
  if (n <= 0) return 0;
  { note_launch(); load_keys_k<<<grid_for(n, 256, sm_count() * 8), 256, 0, st>>>(ks, n, out); }
  return check_launch("load_keys");
}

}  // namespace sfk
