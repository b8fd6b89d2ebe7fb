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
//   * cluster path: when the whole table does not fit one SM but one ROW
//     does (cfg 3/5: a 65536-counter row is 128 KiB as u16), a cluster of d
//     CTAs holds the table row-partitioned in shared memory (CTA r = row r).
//     Each CTA hashes every key of a tile for its own row and gathers locally;
//     the per-row partial counters meet over DSMEM, where CTA r takes the min
//     for its quarter of the tile and stores the int64 estimates. Rows wider
//     than 16 bits are stored clamped to 0xFFFF; a clamped min of 0xFFFF
//     means the true min is >= 65535 and that key re-gathers its d u32
//     counters from global memory, so estimates stay exact.
#include <cooperative_groups.h>

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


namespace cg = cooperative_groups;

// query path override (0 auto, 1 L2, 2 smem, 3 cluster) and the path the last
// launch took, for tests and benchmarks (sfk_query_path / sfk_query_last_path)
static int g_query_path = 0;
static int g_query_last = 0;

int query_path(int mode) {
  int prev = g_query_path;
  if (mode >= 0) g_query_path = mode;
  return prev;
}
int query_last_path() { return g_query_last; }

template <typename CT>
__device__ __forceinline__ CT clamp_ct(uint32_t v) {
  return sizeof(CT) == 2 ? (CT)min(v, 0xFFFFu) : (CT)v;
}

// Vector of 4 counters of type CT (u16 -> 8 B, u32 -> 16 B).
template <typename CT>
struct V4;
template <>
struct V4<uint16_t> {
  using T = uint2;
  __device__ static void unpack(const uint2& v, uint32_t o[4]) {
    o[0] = v.x & 0xFFFFu; o[1] = v.x >> 16; o[2] = v.y & 0xFFFFu; o[3] = v.y >> 16;
  }
  __device__ static uint2 pack(const uint32_t o[4]) { return make_uint2(o[0] | (o[1] << 16), o[2] | (o[3] << 16)); }
};
template <>
struct V4<uint32_t> {
  using T = uint4;
  __device__ static void unpack(const uint4& v, uint32_t o[4]) { o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w; }
  __device__ static uint4 pack(const uint32_t o[4]) { return make_uint4(o[0], o[1], o[2], o[3]); }
};

// One cluster of D CTAs; TILE keys per cluster iteration; NT threads per CTA.
// Shared memory: [row r: w x CT, 16-B padded][partials: 2 x TILE x CT].
template <int D, typename CT, int TILE, int NT>
__global__ void __launch_bounds__(NT, 1) min_query_cluster(const uint32_t* __restrict__ counters, Seeds<D> seeds,
                                                           Mod wm, int64_t w, KeySrc keys, int64_t n,
                                                           int64_t* __restrict__ out, int vec_ok) {
  extern __shared__ uint4 smem_c[];
  cg::cluster_group cl = cg::this_cluster();
  const int r = (int)cl.block_rank();
  CT* row = reinterpret_cast<CT*>(smem_c);
  const size_t row_bytes = ((size_t)w * sizeof(CT) + 15) & ~size_t(15);
  CT* part = reinterpret_cast<CT*>(reinterpret_cast<char*>(smem_c) + row_bytes);
  // stage row r (16-B loads when the row start is aligned)
  const uint32_t* src = counters + (int64_t)r * w;
  int64_t k0 = 0;
  if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
    const int64_t nv = w / 4;
    for (int64_t k = threadIdx.x; k < nv; k += NT) {
      uint4 v = __ldg(reinterpret_cast<const uint4*>(src) + k);
      row[4 * k] = clamp_ct<CT>(v.x); row[4 * k + 1] = clamp_ct<CT>(v.y);
      row[4 * k + 2] = clamp_ct<CT>(v.z); row[4 * k + 3] = clamp_ct<CT>(v.w);
    }
    k0 = nv * 4;
  }
  for (int64_t k = k0 + threadIdx.x; k < w; k += NT) row[k] = clamp_ct<CT>(__ldg(src + k));
  uint64_t seed = seeds.s[0];
#pragma unroll
  for (int i = 1; i < D; ++i)
    if (i == r) seed = seeds.s[i];
  const CT* rpart[D];
#pragma unroll
  for (int i = 0; i < D; ++i) rpart[i] = cl.map_shared_rank(part, i);
  cl.sync();

  const int64_t ntiles = (n + TILE - 1) / TILE;
  const int64_t nclusters = gridDim.x / D;
  constexpr int Q = ((TILE + D - 1) / D + 3) & ~3;  // keys each CTA finalises per tile
  static_assert(TILE % (4 * NT) == 0, "tile shape");
  const int kend = min((r + 1) * Q, TILE);
  const bool u32v = vec_ok && keys.kind == SFK_KEY_U32;
  int it = 0;
  for (int64_t tile = blockIdx.x / D; tile < ntiles; tile += nclusters, ++it) {
    const int64_t base = tile * TILE;
    CT* P = part + (it & 1) * TILE;
    // phase 1: this CTA's row counter for every key of the tile, 4
    // consecutive keys per thread per step (one 16-B key load for u32 keys)
#pragma unroll 2
    for (int k = 4 * threadIdx.x; k < TILE; k += 4 * NT) {
      const int64_t t = base + k;
      uint32_t c[4];
      if (u32v && t + 3 < n) {
        uint4 kk = __ldcs(reinterpret_cast<const uint4*>(static_cast<const uint32_t*>(keys.p) + t));
        c[0] = row[fmod64(mix64((uint64_t)kk.x ^ seed), wm)];
        c[1] = row[fmod64(mix64((uint64_t)kk.y ^ seed), wm)];
        c[2] = row[fmod64(mix64((uint64_t)kk.z ^ seed), wm)];
        c[3] = row[fmod64(mix64((uint64_t)kk.w ^ seed), wm)];
      } else {
#pragma unroll
        for (int u = 0; u < 4; ++u)
          c[u] = (t + u < n) ? (uint32_t)row[fmod64(mix64(load_key(keys, t + u) ^ seed), wm)] : 0u;
      }
      *reinterpret_cast<typename V4<CT>::T*>(P + k) = V4<CT>::pack(c);
    }
    cl.sync();
    // phase 2: min over the D partials for keys [r*Q, (r+1)*Q) of the tile
    const CT* PP[D];
#pragma unroll
    for (int i = 0; i < D; ++i) PP[i] = rpart[i] + (it & 1) * TILE;
    for (int k = r * Q + 4 * threadIdx.x; k < kend; k += 4 * NT) {
      const int64_t t = base + k;
      if (t >= n) break;
      uint32_t m[4], c[4];
      V4<CT>::unpack(*reinterpret_cast<const typename V4<CT>::T*>(PP[0] + k), m);
#pragma unroll
      for (int i = 1; i < D; ++i) {
        V4<CT>::unpack(*reinterpret_cast<const typename V4<CT>::T*>(PP[i] + k), c);
#pragma unroll
        for (int u = 0; u < 4; ++u) m[u] = min(m[u], c[u]);
      }
      if (sizeof(CT) == 2) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (m[u] == 0xFFFFu && t + u < n) {  // true min >= 65535: exact u32 re-gather
            const uint64_t key = load_key(keys, t + u);
            uint32_t mm = U32MAX;
#pragma unroll
            for (int i = 0; i < D; ++i)
              mm = min(mm, __ldg(counters + (int64_t)i * w + (int64_t)fmod64(mix64(key ^ seeds.s[i]), wm)));
            m[u] = mm;
          }
        }
      }
      if (vec_ok && t + 3 < n) {
        longlong2* o2 = reinterpret_cast<longlong2*>(out + t);
        __stcs(o2, make_longlong2((long long)m[0], (long long)m[1]));
        __stcs(o2 + 1, make_longlong2((long long)m[2], (long long)m[3]));
      } else {
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (t + u < n) out[t + u] = (int64_t)m[u];
      }
    }
  }
  cl.sync();  // no CTA may exit while a peer still reads its partials
}

// Launch the cluster kernel if this (d, w, n) suits it; returns -1 if not.
template <int D, typename CT, int TILE>
static int try_cluster(const uint32_t* counters, const Seeds<D>& sd, Mod wm, int64_t w, KeySrc ks, int64_t n,
                       int64_t* out, cudaStream_t st, int optin) {
  constexpr int NT = 1024;
  const size_t row_bytes = ((size_t)w * sizeof(CT) + 15) & ~size_t(15);
  const size_t smem = row_bytes + 2 * (size_t)TILE * sizeof(CT);
  if (smem > (size_t)optin) return -1;
  auto kern = min_query_cluster<D, CT, TILE, NT>;
  static int attr_done = 0;
  if (!attr_done) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, optin) != cudaSuccess) {
      cudaGetLastError();
      return -1;
    }
    attr_done = 1;
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = D;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.gridDim = dim3(D * sm_count());
  int nclusters = 0;
  if (cudaOccupancyMaxActiveClusters(&nclusters, kern, &cfg) != cudaSuccess || nclusters <= 0) {
    cudaGetLastError();
    return -1;
  }
  const int64_t ntiles = (n + TILE - 1) / TILE;
  if ((int64_t)nclusters > ntiles) nclusters = (int)ntiles;
  cfg.gridDim = dim3(D * nclusters);
  const int vec_ok = ((reinterpret_cast<uintptr_t>(out) & 15) == 0) &&
                     (ks.kind != SFK_KEY_U32 || (reinterpret_cast<uintptr_t>(ks.p) & 15) == 0);
  note_launch();
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, counters, sd, wm, w, ks, n, out, vec_ok);
  if (e != cudaSuccess) {
    set_error("min_query_cluster launch: %s", cudaGetErrorString(e));
    return (int)e;
  }
  g_query_last = 3;
  return check_launch("min_query_cluster");
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
  const int mode = g_query_path;
  // staging costs tab_bytes per SM; worth it once the batch's own gathers
  // dwarf it (>= ~16 keys per staged counter word across the chip)
  const bool smem_fits = tab_bytes <= (size_t)optin;
  const bool smem_pays = (double)n * D >= 16.0 * (double)sms * (double)(D * w) / 4.0;
  if ((mode == 0 && smem_fits && smem_pays) || (mode == 2 && smem_fits)) {
    static bool attr_set = false;
    if (!attr_set) {
      cudaFuncSetAttribute(min_query_smem<D, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
      attr_set = true;
    }
    { note_launch(); min_query_smem<D, 4><<<sms, 1024, tab_bytes, st>>>(counters, sd, wm, w, ks, n, out); }
    g_query_last = 2;
    return check_launch("min_query_smem");
  }
  // row-partitioned cluster path: d CTAs per cluster (portable size <= 8);
  // pays once the batch is well beyond the per-CTA row staging (~2M keys)
  if (D >= 2 && D <= 8 && ((mode == 0 && !smem_fits && n >= (int64_t(1) << 21)) || mode == 3)) {
    int rc = -1;
    if ((size_t)w * 4 + 2 * 8192 * 4 + 16 <= (size_t)optin)
      rc = try_cluster<D, uint32_t, 8192>(counters, sd, wm, w, ks, n, out, st, optin);
    else
      rc = try_cluster<D, uint16_t, 16384>(counters, sd, wm, w, ks, n, out, st, optin);
    if (rc >= 0) return rc;
  }
  int blocks = grid_for(n, 256 * 4, sms * 8);
  { note_launch(); min_query_l2<D, 4><<<blocks, 256, 0, st>>>(counters, sd, wm, w, ks, n, out); }
  g_query_last = 1;
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
