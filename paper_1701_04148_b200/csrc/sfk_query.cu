// Batched point query: fused key load + hash + d gathers + min
// (replaces _kernels.min_query, _kernels.py:229-241), plus mix_batch
// (_kernels.py:56-59) and key materialisation.
//
// Three kernels, chosen per call:
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
//     than 16 bits are stored as u16 codes: small values as is, large ones
//     (>= 0xF800, a few hot cells) as their rank among all rows' large values,
//     which the owner decodes from a local table, so estimates stay exact
//     (see OVF_BASE and rank_codes_setup).
#include <cooperative_groups.h>

#include "sfk_common.cuh"

// cluster query kernel shape: threads per CTA and keys per tile (u16 rows)
#ifndef SFK_QUERY_NT
#define SFK_QUERY_NT 512
#endif
#ifndef SFK_QUERY_TILE
#define SFK_QUERY_TILE 8192
#endif

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

// opt-in shared memory per block of the current device (cached per ordinal)
static int smem_optin() {
  static int cache[64];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (cache[dev] <= 0) cudaDeviceGetAttribute(&cache[dev], cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  return cache[dev];
}

// ---- cluster path: PTX helpers (mbarrier, DSMEM st.async) -------------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa_u32(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_arrive(uint32_t a, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
// arrive on a peer CTA's mbarrier. Relaxed: it only signals that this CTA's
// reads of a receive buffer are done, and those reads have already returned
// (their values were consumed before the __syncthreads preceding the arrive);
// a .release arrive would cost a GPU-scope MEMBAR per tile.
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done) : "r"(a), "r"(parity) : "memory");
  } while (!done);
}
// asynchronous remote store that completes `bytes` of the peer's mbarrier tx
__device__ __forceinline__ void st_async_v2(uint32_t cluster_addr, uint32_t a, uint32_t b, uint32_t cluster_mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b32 [%0], {%1, %2}, [%3];" ::"r"(cluster_addr),
               "r"(a), "r"(b), "r"(cluster_mbar) : "memory");
}
__device__ __forceinline__ void st_async_v4(uint32_t cluster_addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d,
                                            uint32_t cluster_mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                   cluster_addr), "r"(a), "r"(b), "r"(c), "r"(d), "r"(cluster_mbar) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Row index for the cluster kernel: the low 32 bits of finalize64(key ^ seed)
// suffice for a power-of-two width (x ^ (x >> 31) masked), else the exact
// 64-bit reduction.
template <bool POW2>
__device__ __forceinline__ uint32_t row_index(uint64_t key, uint64_t seed, const Mod& M) {
  if (POW2) {
    uint64_t x = key ^ seed;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return ((uint32_t)x ^ (uint32_t)(x >> 31)) & (uint32_t)M.mask;
  }
  return (uint32_t)fmod64(mix64(key ^ seed), M);
}

// finalize64(key ^ seed) mod 2^k for a 32-bit key, in 32-bit halves: the
// high word of key ^ seed is the seed's, so the first xor-shift's high half
// and its share of the first multiply are per-CTA constants (U32Hash).
struct U32Hash {
  uint32_t slo;  // low word of the seed
  uint32_t c1;   // seed_hi << 2: the high bits shifted into the low word by x >> 30
  uint32_t c2;   // (seed_hi ^ seed_hi >> 30) * lo32(K1): the high-word term of x * K1
};
__host__ __device__ __forceinline__ U32Hash make_u32hash(uint64_t seed) {
  const uint32_t hi = (uint32_t)(seed >> 32);
  return U32Hash{(uint32_t)seed, hi << 2, (hi ^ (hi >> 30)) * 0x1CE4E5B9u};
}
__device__ __forceinline__ uint32_t row_index_u32(uint32_t key, const U32Hash& h, uint32_t mask) {
  const uint32_t lo = key ^ h.slo;
  const uint32_t lo1 = lo ^ (lo >> 30) ^ h.c1;
  // x *= 0xBF58476D1CE4E5B9
  const uint64_t w1 = (uint64_t)lo1 * 0x1CE4E5B9u + ((uint64_t)h.c2 << 32);
  const uint32_t lo2 = (uint32_t)w1, hi2 = (uint32_t)(w1 >> 32) + lo1 * 0xBF58476Du;
  // x ^= x >> 27
  const uint32_t lo3 = lo2 ^ __funnelshift_r(lo2, hi2, 27), hi3 = hi2 ^ (hi2 >> 27);
  // x *= 0x94D049BB133111EB
  const uint64_t w2 = (uint64_t)lo3 * 0x133111EBu;
  const uint32_t lo4 = (uint32_t)w2, hi4 = (uint32_t)(w2 >> 32) + lo3 * 0x94D049BBu + hi3 * 0x133111EBu;
  // low word of x ^ (x >> 31)
  return (lo4 ^ __funnelshift_r(lo4, hi4, 31)) & mask;
}

// u16 row encoding: values below OVF_BASE are stored as is; a larger value
// gets the code OVF_BASE + s and its exact u32 value in overflow slot s of
// its row; OVF_NONE marks a large value that found no slot (re-read from
// global memory). Codes order below every large value, so a min over codes
// that is < OVF_BASE is the exact min. At setup the codes become ranks among
// all rows' large values (a few hot cells), so decoding is one local load.
constexpr uint32_t OVF_BASE = 0xF800u;
constexpr uint32_t OVF_NONE = 0xFFFFu;
constexpr int OVF_SLOTS = (int)(OVF_NONE - OVF_BASE);  // 2047 per row
constexpr int OVF_STRIDE = OVF_SLOTS + 1;               // + the slot count
constexpr int QNB = 2;                                 // receive buffers per CTA

// internal key kind: precomputed u16 row indices (sfk_query_index), row r's
// stream at p + r * n
constexpr int KEY_IDX16 = 3;

template <int KK>
__device__ __forceinline__ uint64_t key_at(const KeySrc& k, int64_t t) {
  if (KK == SFK_KEY_U32) return (uint64_t)__ldg(static_cast<const unsigned int*>(k.p) + t);
  if (KK == SFK_KEY_U64) return __ldg(static_cast<const unsigned long long*>(k.p) + t);
  return record_key(static_cast<const uint8_t*>(k.p) + t * (int64_t)k.rec, k.rec);
}

// Setup of the u16 rank codes (kept out of line so it does not perturb the
// main loop's register allocation): rank every large value among all rows'
// large values (read over DSMEM) and re-encode this row's codes as
// OVF_BASE + rank; codes then order like the values across rows, so the
// owner decodes only the minimum code, with one local load. Exhausted
// tables keep per-row slot codes. Returns whether the rank codes apply.
template <int D, typename CT, int NT>
__device__ __noinline__ int rank_codes_setup(CT* row, uint32_t* ovf, uint32_t* merged, uint32_t* own_rank, int64_t w,
                                             uint32_t r) {
  const uint32_t* tab[D];
  int cnt[D], total = 0;
  bool ok = true;
#pragma unroll
  for (int q = 0; q < D; ++q) {
    tab[q] = cg::this_cluster().map_shared_rank(ovf, q);
    const int raw = (int)tab[q][OVF_SLOTS];
    ok = ok && raw <= OVF_SLOTS;
    cnt[q] = min(raw, OVF_SLOTS);
    total += cnt[q];
  }
  ok = ok && total <= OVF_SLOTS;
  if (ok) {
    for (int idx = threadIdx.x; idx < total; idx += NT) {
      int q = 0, s = idx;
#pragma unroll
      for (int qq = 0; qq < D - 1; ++qq)
        if (s >= cnt[q]) s -= cnt[q], ++q;
      const uint32_t v = tab[q][s];
      int rank = 0;
#pragma unroll 1
      for (int q2 = 0; q2 < D; ++q2)
        for (int s2 = 0; s2 < cnt[q2]; ++s2) rank += tab[q2][s2] < v;
      merged[rank] = v;
      if (q == (int)r) own_rank[s] = (uint32_t)rank;
    }
    __syncthreads();
    for (int64_t k = threadIdx.x; k < w; k += NT) {
      const uint32_t cde = row[k];
      if (cde >= OVF_BASE && cde != OVF_NONE) row[k] = (CT)(OVF_BASE + own_rank[cde - OVF_BASE]);
    }
  } else {
    // exhausted: every large value re-reads its u32 counter from global memory
    __syncthreads();
    for (int64_t k = threadIdx.x; k < w; k += NT)
      if ((uint32_t)row[k] >= OVF_BASE) row[k] = (CT)OVF_NONE;
  }
  return ok ? 1 : 0;
}

// Row-partitioned cluster query. A cluster of D CTAs; CTA r holds slim row r
// in shared memory. Per tile of TILE keys (the cluster's tiles are strided
// over the grid's clusters):
//   phase 1 (every CTA): row-r counter of each key; the partials of the keys
//     CTA q owns (the q-th 1/D of the tile) go to CTA q's receive buffer with
//     st.async, which completes bytes on CTA q's `full` mbarrier;
//   phase 2 (owner q, one tile behind phase 1 so the transfers overlap the
//     hashing): wait `full`, min over the D partials, decode large values,
//     int64 stores; then release the buffer with a remote arrive on every
//     producer's `empty` mbarrier.
// Shared memory: [row: w x CT][overflow: D x OVF_STRIDE u32, u16 rows only]
// [recv: QNB x D x Q x CT][mbarriers: full[QNB], empty[QNB]].
template <int D, typename CT, int TILE, int NT, int KK, bool VEC, bool POW2>
__global__ void __launch_bounds__(NT, 1) min_query_cluster(const uint32_t* __restrict__ counters, Seeds<D> seeds,
                                                           Mod wm, int64_t w, KeySrc keys, int64_t n,
                                                           int64_t* __restrict__ out, int out_vec) {
  constexpr bool U16 = sizeof(CT) == 2;
  constexpr int KPT = TILE / NT;  // keys per thread per tile (phase 1)
  constexpr int VPT = KPT / 4;    // 4-key groups per thread
  constexpr int Q = ((TILE + D - 1) / D + 3) & ~3;
  static_assert(TILE % (4 * NT) == 0, "tile shape");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t r = cg::this_cluster().block_rank();
  CT* row = reinterpret_cast<CT*>(smem_raw);
  const size_t row_bytes = ((size_t)w * sizeof(CT) + 15) & ~size_t(15);
  // u16 rows: this row's overflow table (values + count, read by the peers
  // during setup) and the cluster-wide rank table (rank -> value)
  uint32_t* ovf = reinterpret_cast<uint32_t*>(smem_raw + row_bytes);
  uint32_t* merged = ovf + OVF_STRIDE;
  CT* recv = reinterpret_cast<CT*>(smem_raw + row_bytes + (U16 ? 2 * OVF_STRIDE * 4 : 0));
  uint32_t* my_ovf = ovf;
  int& novf = *reinterpret_cast<int*>(my_ovf + OVF_SLOTS);
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(recv + (size_t)QNB * D * Q);
  // bars[0..QNB) = full, bars[QNB..2QNB) = empty
  if (threadIdx.x == 0) {
    novf = 0;
    for (int b = 0; b < QNB; ++b) {
      mbar_init(smem_addr(bars + b), 1);
      mbar_init(smem_addr(bars + QNB + b), D);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // stage row r (u16 rows: large values into the overflow slots)
  const uint32_t* src = counters + (int64_t)r * w;
  for (int64_t k = threadIdx.x; k < w; k += NT) {
    uint32_t v = __ldg(src + k);
    if (U16 && v >= OVF_BASE) {
      int s = atomicAdd(&novf, 1);
      if (s < OVF_SLOTS) {
        my_ovf[s] = v;
        v = OVF_BASE + (uint32_t)s;
      } else {
        v = OVF_NONE;
      }
    }
    row[k] = (CT)v;
  }
  uint64_t seed = seeds.s[0];
#pragma unroll
  for (int i = 1; i < D; ++i)
    if (i == (int)r) seed = seeds.s[i];
  const U32Hash h32 = make_u32hash(seed);
  const uint32_t mask32 = (uint32_t)wm.mask;
  const uint32_t recv_a = smem_addr(recv), bars_a = smem_addr(bars);
  uint32_t peer_recv[D], peer_full[D];
#pragma unroll
  for (int q = 0; q < D; ++q) {
    peer_recv[q] = mapa_u32(recv_a, q);
    peer_full[q] = mapa_u32(bars_a, q);
  }
  cluster_sync_all();  // rows staged, barriers initialised cluster-wide
  if (U16) {
    (void)rank_codes_setup<D, CT, NT>(row, ovf, merged, reinterpret_cast<uint32_t*>(recv), w, r);
    cluster_sync_all();  // peers done reading this table; recv scratch free
  }

  const int64_t ntiles = (n + TILE - 1) / TILE;
  const int64_t nclusters = gridDim.x / D;
  const int64_t cid = blockIdx.x / D;
  const int64_t T = cid < ntiles ? (ntiles - 1 - cid) / nclusters + 1 : 0;  // tiles of this cluster
  const int own_lo = (int)r * Q, own_hi = min(((int)r + 1) * Q, TILE);
  const int owned = max(own_hi - own_lo, 0);
  const uint32_t* k32 = static_cast<const uint32_t*>(keys.p);

  uint4 kn[VEC ? VPT : 1];
  const uint16_t* i16 = KK == KEY_IDX16 ? static_cast<const uint16_t*>(keys.p) + (int64_t)r * n : nullptr;
  auto prefetch = [&](int64_t it) {
    if (VEC && KK == KEY_IDX16 && it < T) {  // four u16 row indices per 8-B load
      const int64_t base = (cid + it * nclusters) * TILE;
      const uint2* src2 = reinterpret_cast<const uint2*>(i16 + base) + threadIdx.x;
#pragma unroll
      for (int j = 0; j < VPT; ++j) {
        const int64_t t = base + 4 * threadIdx.x + (int64_t)j * 4 * NT;
        const uint2 v = (t + 3 < n) ? __ldcs(src2 + j * NT) : make_uint2(0, 0);
        kn[j] = make_uint4(v.x, v.y, 0, 0);
      }
    } else if (VEC && it < T) {
      const int64_t base = (cid + it * nclusters) * TILE;
      const uint4* src4 = reinterpret_cast<const uint4*>(k32 + base) + threadIdx.x;
      if (base + TILE <= n) {
#pragma unroll
        for (int j = 0; j < VPT; ++j) kn[j] = __ldcs(src4 + j * NT);
      } else {
#pragma unroll
        for (int j = 0; j < VPT; ++j) {
          const int64_t t = base + 4 * threadIdx.x + (int64_t)j * 4 * NT;
          kn[j] = (t + 3 < n) ? __ldcs(src4 + j * NT) : make_uint4(0, 0, 0, 0);
        }
      }
    }
  };
  prefetch(0);

  for (int64_t i = 0; i <= T; ++i) {
    if (i < T) {
      // ---------------- phase 1: tile i into buffer i % QNB of every owner
      const int b = (int)(i % QNB);
      if (threadIdx.x == 0) mbar_expect_arrive(bars_a + b * 8, (uint32_t)(D * owned * sizeof(CT)));
      if (i >= QNB) mbar_wait(bars_a + (QNB + b) * 8, (uint32_t)((i / QNB - 1) & 1));  // owners released it
      const int64_t base = (cid + i * nclusters) * TILE;
      uint4 kk[VEC ? VPT : 1];
      if (VEC) {
#pragma unroll
        for (int j = 0; j < VPT; ++j) kk[j] = kn[j];
        prefetch(i + 1);
      }
      // all VPT x 4 row counters first (independent hash chains and smem
      // gathers in flight together), then the D-way scatter with st.async
      uint32_t c[VPT][4];
      if (VEC && base + TILE <= n) {
#pragma unroll
        for (int j = 0; j < VPT; ++j) {
          if (KK == KEY_IDX16) {
            c[j][0] = row[kk[j].x & 0xFFFFu];
            c[j][1] = row[kk[j].x >> 16];
            c[j][2] = row[kk[j].y & 0xFFFFu];
            c[j][3] = row[kk[j].y >> 16];
            continue;
          }
          c[j][0] = row[POW2 ? row_index_u32(VEC ? kk[j].x : 0u, h32, mask32) : row_index<POW2>(VEC ? kk[j].x : 0u, seed, wm)];
          c[j][1] = row[POW2 ? row_index_u32(VEC ? kk[j].y : 0u, h32, mask32) : row_index<POW2>(VEC ? kk[j].y : 0u, seed, wm)];
          c[j][2] = row[POW2 ? row_index_u32(VEC ? kk[j].z : 0u, h32, mask32) : row_index<POW2>(VEC ? kk[j].z : 0u, seed, wm)];
          c[j][3] = row[POW2 ? row_index_u32(VEC ? kk[j].w : 0u, h32, mask32) : row_index<POW2>(VEC ? kk[j].w : 0u, seed, wm)];
        }
      } else {
#pragma unroll
        for (int j = 0; j < VPT; ++j) {
          const int64_t t = base + 4 * threadIdx.x + j * 4 * NT;
#pragma unroll
          for (int u = 0; u < 4; ++u)
            c[j][u] = (t + u < n) ? (KK == KEY_IDX16 ? (uint32_t)row[i16[t + u]]
                                                     : (uint32_t)row[row_index<POW2>(key_at<KK>(keys, t + u), seed, wm)])
                                  : 0u;
        }
      }
#pragma unroll
      for (int j = 0; j < VPT; ++j) {
        const int k = 4 * threadIdx.x + j * 4 * NT;
        // owner of keys k .. k+3 (Q is a multiple of 4); compile-time when
        // each thread's 4-key groups map one-to-one onto the D owners
        const int q = (Q == 4 * NT) ? j : k / Q;
        uint32_t qa = 0, qb = 0;
#pragma unroll
        for (int p = 0; p < D; ++p)
          if (p == q) qa = peer_recv[p], qb = peer_full[p];
        const uint32_t off = (uint32_t)((((size_t)b * D + r) * Q + (k - q * Q)) * sizeof(CT));
        if (U16)
          st_async_v2(qa + off, c[j][0] | (c[j][1] << 16), c[j][2] | (c[j][3] << 16), qb + b * 8);
        else
          st_async_v4(qa + off, c[j][0], c[j][1], c[j][2], c[j][3], qb + b * 8);
      }
    }
    if (i >= 1) {
      // ---------------- phase 2: tile i-1 from buffer (i-1) % QNB
      const int64_t ip = i - 1;
      const int b = (int)(ip % QNB);
      mbar_wait(bars_a + b * 8, (uint32_t)((ip / QNB) & 1));
      const int64_t base = (cid + ip * nclusters) * TILE + own_lo;
      const CT* R = recv + (size_t)b * D * Q;
      for (int k = 4 * threadIdx.x; k < owned; k += 4 * NT) {
        const int64_t t = base + k;
        if (t >= n) break;
        uint32_t cc[D][4], m[4];
#pragma unroll
        for (int p = 0; p < D; ++p) {
          if (U16) {
            const uint2 v = *reinterpret_cast<const uint2*>(R + (size_t)p * Q + k);
            cc[p][0] = v.x & 0xFFFFu; cc[p][1] = v.x >> 16; cc[p][2] = v.y & 0xFFFFu; cc[p][3] = v.y >> 16;
          } else {
            const uint4 v = *reinterpret_cast<const uint4*>(R + (size_t)p * Q + k);
            cc[p][0] = v.x; cc[p][1] = v.y; cc[p][2] = v.z; cc[p][3] = v.w;
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          m[u] = cc[0][u];
#pragma unroll
          for (int p = 1; p < D; ++p) m[u] = min(m[u], cc[p][u]);
        }
        if (U16) {
          // codes below OVF_NONE are ranks across all rows: the minimum code
          // decodes alone; OVF_NONE (overflow tables exhausted) re-reads the
          // key's d u32 counters
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (m[u] >= OVF_BASE) {
              if (m[u] != OVF_NONE) {
                m[u] = merged[m[u] - OVF_BASE];
              } else if (t + u < n) {
                uint32_t mm = U32MAX;
                if (KK == KEY_IDX16) {
                  const uint16_t* ix = static_cast<const uint16_t*>(keys.p);
#pragma unroll
                  for (int p = 0; p < D; ++p) mm = min(mm, __ldg(counters + (int64_t)p * w + ix[(int64_t)p * n + t + u]));
                } else {
                  const uint64_t key = key_at<KK>(keys, t + u);
#pragma unroll
                  for (int p = 0; p < D; ++p)
                    mm = min(mm, __ldg(counters + (int64_t)p * w + (int64_t)fmod64(mix64(key ^ seeds.s[p]), wm)));
                }
                m[u] = mm;
              }
            }
          }
        }
        if (out_vec && t + 3 < n) {
          longlong2* o2 = reinterpret_cast<longlong2*>(out + t);
          __stcs(o2, make_longlong2((long long)m[0], (long long)m[1]));
          __stcs(o2 + 1, make_longlong2((long long)m[2], (long long)m[3]));
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (t + u < n) out[t + u] = (int64_t)m[u];
        }
      }
      // release the buffer to every producer, unless nobody will refill it
      if (ip + QNB < T) {
        __syncthreads();
        if (threadIdx.x < D) mbar_arrive_remote(mapa_u32(bars_a + (QNB + b) * 8, threadIdx.x));
      }
    }
  }
  cluster_sync_all();  // no CTA exits while peers may still touch its shared memory
}

// warp-pipelined kernel shape (A/B knobs): warps per CTA, keys per lane per
// tile (d = 4; d = 2 uses 8, d = 8 uses 16), receive buffers per warp
#ifndef SFK_CW_NW
#define SFK_CW_NW 16
#endif
#ifndef SFK_CW_KPL
#define SFK_CW_KPL 16
#endif
#ifndef SFK_CW_NB
#define SFK_CW_NB 4
#endif

// ---- cluster path, warp-pipelined (u32 keys) ---------------------------------
// Same row partition as min_query_cluster (CTA r of a D-CTA cluster holds slim
// row r in shared memory), but the exchange runs per warp instead of per CTA:
// warp w of every CTA of the cluster forms a "group" that works through its
// own sequence of K-key warp-tiles, coupled only by per-warp mbarriers, so
// there is no CTA-wide barrier in the steady state and warps hide each other's
// latencies. Per warp-tile:
//   keys   : every lane loads its KPL keys of the next tile into registers
//            (LDG.128) one tile ahead (a TMA key ring in shared memory measured
//            slower: it forces a smaller tile, and the tile size is what
//            amortises the per-tile synchronisation);
//   phase 1: every lane hashes KPL keys for row r and gathers their codes;
//            4-key group gk goes to the CTA owning its 1/D of the tile with
//            one st.async that completes bytes on the owner's `full` mbarrier;
//   phase 2: one tile behind, the owner takes the min over the D partials
//            (packed u16x2 VIMNMX), decodes rank codes and stores int64s;
//            then it releases the buffer with a remote arrive on every
//            producer's `empty` mbarrier.

// finalize64(key ^ seed) for a 32-bit key, reduced to the BYTE offset of its
// cell in a power-of-two row of 2^SH-byte codes: (idx << SH) comes straight
// out of x' = x << SH (the second multiply by K2 << SH), so no extra shift.
// v = u ^ u >> 30 with u = key ^ seed: the low word is key ^ (key >> 30) ^ c0.
struct U32HashOff {
  uint32_t c0;  // s_lo ^ (s_lo >> 30) ^ (s_hi << 2)
  uint32_t c2;  // lo32((s_hi ^ s_hi >> 30) * lo32(K1)): the high-word term of v * K1
};
__host__ __device__ __forceinline__ U32HashOff make_u32hash_off(uint64_t seed) {
  const uint32_t lo = (uint32_t)seed, hi = (uint32_t)(seed >> 32);
  return U32HashOff{lo ^ (lo >> 30) ^ (hi << 2), (hi ^ (hi >> 30)) * 0x1CE4E5B9u};
}
// Written in PTX so that ptxas keeps the short form (15 per key and row with
// the shift of k30 and the gather): one 3-input LOP3 for v, the first product
// as three FMA-pipe IMADs (lo, hi + the seed's high-word term, hi word of
// K1), two funnel/xor pairs, IMAD.WIDE + 2 IMAD, and the final
// (x ^ x >> 31) & mask as one SHF + one LOP3. (From C++ the compiler
// re-associates v through key ^ seed and adds a carry chain: ~17.5.)
// k30 = key >> 30.
template <int SH>
__device__ __forceinline__ uint32_t row_off_u32(uint32_t key, uint32_t k30, uint32_t c0, uint32_t c2, uint32_t mask_b) {
  constexpr uint64_t K2S = 0x94D049BB133111EBull << SH;
  uint32_t r;
  asm("{\n\t"
      ".reg .b32 v, zl, zh, t, yl, yh, xl, xh;\n\t"
      ".reg .b64 x;\n\t"
      "lop3.b32 v, %1, %2, %3, 0x96;\n\t"
      "mul.lo.u32 zl, v, 0x1CE4E5B9;\n\t"
      "mad.hi.u32 zh, v, 0x1CE4E5B9, %4;\n\t"
      "mad.lo.u32 zh, v, 0xBF58476D, zh;\n\t"
      "shf.r.wrap.b32 t, zl, zh, 27;\n\t"
      "xor.b32 yl, zl, t;\n\t"
      "shr.u32 t, zh, 27;\n\t"
      "xor.b32 yh, zh, t;\n\t"
      "mul.wide.u32 x, yl, %6;\n\t"
      "mov.b64 {xl, xh}, x;\n\t"
      "mad.lo.u32 xh, yl, %7, xh;\n\t"
      "mad.lo.u32 xh, yh, %6, xh;\n\t"
      "shf.r.wrap.b32 t, xl, xh, 31;\n\t"
      "lop3.b32 %0, xl, t, %5, 0x28;\n\t"
      "}"
      : "=r"(r)
      : "r"(key), "r"(k30), "r"(c0), "r"(c2), "r"(mask_b), "n"((uint32_t)K2S), "n"((uint32_t)(K2S >> 32)));
  return r;
}

// The same reduction for a 64-bit key (the reference's own key dtype): the
// high word of key ^ seed is no longer a per-CTA constant, so v and the first
// product take the full 64-bit form (17 instructions per key and row).
template <int SH>
__device__ __forceinline__ uint32_t row_off_u64(uint32_t klo, uint32_t khi, uint32_t slo, uint32_t shi,
                                                uint32_t mask_b) {
  constexpr uint64_t K2S = 0x94D049BB133111EBull << SH;
  uint32_t r;
  asm("{\n\t"
      ".reg .b32 ul, uh, vl, vh, zl, zh, t, yl, yh, xl, xh;\n\t"
      ".reg .b64 x;\n\t"
      "xor.b32 ul, %1, %3;\n\t"
      "xor.b32 uh, %2, %4;\n\t"
      "shf.r.wrap.b32 t, ul, uh, 30;\n\t"
      "xor.b32 vl, ul, t;\n\t"
      "shr.u32 t, uh, 30;\n\t"
      "xor.b32 vh, uh, t;\n\t"
      "mul.lo.u32 zl, vl, 0x1CE4E5B9;\n\t"
      "mul.hi.u32 zh, vl, 0x1CE4E5B9;\n\t"
      "mad.lo.u32 zh, vl, 0xBF58476D, zh;\n\t"
      "mad.lo.u32 zh, vh, 0x1CE4E5B9, zh;\n\t"
      "shf.r.wrap.b32 t, zl, zh, 27;\n\t"
      "xor.b32 yl, zl, t;\n\t"
      "shr.u32 t, zh, 27;\n\t"
      "xor.b32 yh, zh, t;\n\t"
      "mul.wide.u32 x, yl, %6;\n\t"
      "mov.b64 {xl, xh}, x;\n\t"
      "mad.lo.u32 xh, yl, %7, xh;\n\t"
      "mad.lo.u32 xh, yh, %6, xh;\n\t"
      "shf.r.wrap.b32 t, xl, xh, 31;\n\t"
      "lop3.b32 %0, xl, t, %5, 0x28;\n\t"
      "}"
      : "=r"(r)
      : "r"(klo), "r"(khi), "r"(slo), "r"(shi), "r"(mask_b), "n"((uint32_t)K2S), "n"((uint32_t)(K2S >> 32)));
  return r;
}

// KU64: 64-bit keys (else u32)
template <int D, typename CT, int NW, int KPL, int NB, bool POW2, bool KU64>
__global__ void __launch_bounds__(NW * 32, 1) min_query_cw(const uint32_t* __restrict__ counters, Seeds<D> seeds,
                                                           Mod wm, int64_t w, const void* __restrict__ keys_v,
                                                           int64_t ntiles, int64_t* __restrict__ out) {
  constexpr bool U16 = sizeof(CT) == 2;
  constexpr int SH = U16 ? 1 : 2;
  constexpr int NT = NW * 32;
  constexpr int KW = KU64 ? 2 : 1;  // 32-bit words per key
  constexpr int K = 32 * KPL;              // keys per warp-tile
  constexpr int OKL = KPL / D;             // keys per lane in the owner phase
  constexpr uint32_t RB = K * sizeof(CT);  // receive bytes per (warp, buffer)
  constexpr uint32_t PB = RB / D;          // one producer's share
  constexpr uint32_t GB = 4 * sizeof(CT);  // bytes of one 4-key group of codes
  static_assert(KPL % 4 == 0 && (OKL == 2 || OKL == 4) && 32 % D == 0 && (NB == 2 || NB == 4), "tile shape");
  constexpr int LNB = NB == 2 ? 1 : 2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t r = cg::this_cluster().block_rank();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  CT* row = reinterpret_cast<CT*>(smem_raw);
  const size_t row_bytes = ((size_t)w * sizeof(CT) + 15) & ~size_t(15);
  uint32_t* ovf = reinterpret_cast<uint32_t*>(smem_raw + row_bytes);
  uint32_t* merged = ovf + OVF_STRIDE;
  unsigned char* recv = smem_raw + row_bytes + (U16 ? 2 * OVF_STRIDE * 4 : 0);  // NW x NB x RB
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(recv + (size_t)NW * NB * RB);
  // per warp: full[NB] (count 1), empty[NB] (count D)
  constexpr int NBAR = 2 * NB;
  int& novf = *reinterpret_cast<int*>(ovf + OVF_SLOTS);
  if (threadIdx.x == 0) novf = 0;
  if (threadIdx.x < NW) {
    unsigned long long* b = bars + threadIdx.x * NBAR;
    for (int k = 0; k < NB; ++k) mbar_init(smem_addr(b + k), 1);
    for (int k = 0; k < NB; ++k) mbar_init(smem_addr(b + NB + k), D);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t* src = counters + (int64_t)r * w;
  for (int64_t k = threadIdx.x; k < w; k += NT) {
    uint32_t v = __ldg(src + k);
    if (U16 && v >= OVF_BASE) {
      const int s = atomicAdd(&novf, 1);
      if (s < OVF_SLOTS) {
        ovf[s] = v;
        v = OVF_BASE + (uint32_t)s;
      } else {
        v = OVF_NONE;
      }
    }
    row[k] = (CT)v;
  }
  cluster_sync_all();
  if (U16) {
    (void)rank_codes_setup<D, CT, NT>(row, ovf, merged, reinterpret_cast<uint32_t*>(recv), w, r);
    if (threadIdx.x == 0) merged[OVF_SLOTS] = U32MAX;  // OVF_NONE decodes to the re-read sentinel
    cluster_sync_all();
  }

  uint64_t seed = seeds.s[0];
#pragma unroll
  for (int i = 1; i < D; ++i)
    if (i == (int)r) seed = seeds.s[i];
  const U32HashOff hh = make_u32hash_off(seed);
  const uint32_t mask_b = (uint32_t)wm.mask << SH;
  const int64_t ncl = gridDim.x / D, cid = blockIdx.x / D;
  const int64_t g0 = cid * NW + warp, gstride = ncl * NW;
  const int Tw = g0 < ntiles ? (int)((ntiles - 1 - g0) / gstride + 1) : 0;
  const int64_t tstep = gstride * K;  // key offset between a warp's consecutive tiles
  const uint32_t rv_a = smem_addr(recv + (size_t)warp * NB * RB);
  const uint32_t bar_a = smem_addr(bars + warp * NBAR);
  const uint32_t full_a = bar_a, empty_a = bar_a + 8 * NB;
  // 4-key group gk = 32 j + lane of a tile goes to owner CTA gk / GD (each
  // owner takes a contiguous 1/D of the tile, so its int64 stores coalesce),
  // slot gk % GD of producer r's share
  constexpr int GD = K / 4 / D;
  uint32_t o_recv[KPL / 4], o_full[KPL / 4];
#pragma unroll
  for (int j = 0; j < KPL / 4; ++j) {
    const int gk = 32 * j + lane;
    o_recv[j] = mapa_u32(rv_a, (uint32_t)(gk / GD)) + r * PB + (uint32_t)(gk % GD) * GB;
    o_full[j] = mapa_u32(full_a, (uint32_t)(gk / GD));
  }
  const uint32_t p_empty = mapa_u32(empty_a, (uint32_t)(lane < D ? lane : 0));

  // owner phase of tile ip (keys from tile_key) in receive buffer pb
  auto owner_phase = [&](int ip, int pb, uint32_t par, int64_t tile_key) {
    mbar_wait(full_a + 8 * pb, par);
    // the owner's 1/D of the tile: OKL consecutive keys per lane, at byte
    // lane * OKL * sizeof(CT) of every producer's share
    const int64_t t = tile_key + (int64_t)r * (K / D) + lane * OKL;
    uint32_t m[OKL];
    const unsigned char* R = recv + ((size_t)warp * NB + pb) * RB;
    if constexpr (U16) {
      uint32_t pk[OKL / 2];
#pragma unroll
      for (int p = 0; p < D; ++p) {
        uint32_t v[OKL / 2];
        if constexpr (OKL == 2) {
          v[0] = *reinterpret_cast<const uint32_t*>(R + p * PB + lane * 4);
        } else {
          const uint2 q2 = *reinterpret_cast<const uint2*>(R + p * PB + lane * 8);
          v[0] = q2.x;
          v[OKL / 2 - 1] = q2.y;
        }
#pragma unroll
        for (int u = 0; u < OKL / 2; ++u) pk[u] = p == 0 ? v[u] : __vminu2(pk[u], v[u]);
      }
#pragma unroll
      for (int u = 0; u < OKL / 2; ++u) m[2 * u] = pk[u] & 0xFFFFu, m[2 * u + 1] = pk[u] >> 16;
      // rank codes decode with one (predicated) table load each; OVF_NONE
      // maps to the U32MAX sentinel in merged[OVF_SLOTS], and only a U32MAX
      // result (exhausted tables, or a counter that really is U32MAX)
      // re-reads the key's d u32 counters
      bool big = false;
#pragma unroll
      for (int u = 0; u < OKL; ++u) big |= m[u] >= OVF_BASE;
      bool none = false;
      if (__any_sync(0xFFFFFFFFu, big)) {  // warp-uniform: no divergence on Zipf-hot tiles
#pragma unroll
        for (int u = 0; u < OKL; ++u) {
          if (m[u] >= OVF_BASE) m[u] = merged[m[u] - OVF_BASE];
          none |= m[u] == U32MAX;
        }
      }
      if (none) {
#pragma unroll
        for (int u = 0; u < OKL; ++u) {
          if (m[u] == U32MAX) {
            const uint64_t key = KU64 ? __ldg(static_cast<const unsigned long long*>(keys_v) + t + u)
                                      : (uint64_t)__ldg(static_cast<const uint32_t*>(keys_v) + t + u);
            uint32_t mm = U32MAX;
#pragma unroll
            for (int p = 0; p < D; ++p)
              mm = min(mm, __ldg(counters + (int64_t)p * w + (int64_t)fmod64(mix64(key ^ seeds.s[p]), wm)));
            m[u] = mm;
          }
        }
      }
    } else {
#pragma unroll
      for (int p = 0; p < D; ++p) {
        uint32_t v[OKL];
        if constexpr (OKL == 2) {
          const uint2 q2 = *reinterpret_cast<const uint2*>(R + p * PB + lane * 8);
          v[0] = q2.x;
          v[OKL - 1] = q2.y;
        } else {
          const uint4 q4 = *reinterpret_cast<const uint4*>(R + p * PB + lane * 16);
          v[0] = q4.x;
          v[1] = q4.y;
          v[OKL - 2] = q4.z;
          v[OKL - 1] = q4.w;
        }
#pragma unroll
        for (int u = 0; u < OKL; ++u) m[u] = p == 0 ? v[u] : min(m[u], v[u]);
      }
    }
    longlong2* o2 = reinterpret_cast<longlong2*>(out + t);
#pragma unroll
    for (int u = 0; u < OKL / 2; ++u) __stcs(o2 + u, make_longlong2((long long)m[2 * u], (long long)m[2 * u + 1]));
    __syncwarp();
    if (ip + NB < Tw && lane < D) mbar_arrive_remote(p_empty + 8 * pb);
  };

  // NB receive buffers (a power of two): buffer and phase parity are bits of
  // the tile counter
  int64_t tile_key = g0 * K;
  uint4 kn[KW * KPL / 4];  // the next tile's keys (4-key group j*32 + lane: KW uint4s)
  auto gload = [&](int64_t tk) {
    const uint4* src = reinterpret_cast<const uint4*>(static_cast<const uint32_t*>(keys_v) + tk * KW) + lane * KW;
#pragma unroll
    for (int j = 0; j < KPL / 4; ++j)
#pragma unroll
      for (int h = 0; h < KW; ++h) kn[KW * j + h] = __ldcs(src + j * 32 * KW + h);
  };
  if (Tw > 0) gload(tile_key);
  for (int it = 0; it < Tw; ++it) {
    const int pb = it & (NB - 1);
    uint4 kk[KW * KPL / 4];
#pragma unroll
    for (int j = 0; j < KW * KPL / 4; ++j) kk[j] = kn[j];
    if (it + 1 < Tw) gload(tile_key + tstep);
    if (lane == 0) mbar_expect_arrive(full_a + 8 * pb, RB);
    uint32_t c[KPL];
    const unsigned char* rowb = reinterpret_cast<const unsigned char*>(row);
#pragma unroll
    for (int j = 0; j < KPL / 4; ++j) {
      uint32_t klo[4], khi[4];
      if constexpr (KU64) {
        klo[0] = kk[2 * j].x, khi[0] = kk[2 * j].y, klo[1] = kk[2 * j].z, khi[1] = kk[2 * j].w;
        klo[2] = kk[2 * j + 1].x, khi[2] = kk[2 * j + 1].y, klo[3] = kk[2 * j + 1].z, khi[3] = kk[2 * j + 1].w;
      } else {
        klo[0] = kk[j].x, klo[1] = kk[j].y, klo[2] = kk[j].z, klo[3] = kk[j].w;
        khi[0] = khi[1] = khi[2] = khi[3] = 0u;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        uint32_t off;
        if constexpr (POW2 && KU64)
          off = row_off_u64<SH>(klo[u], khi[u], (uint32_t)seed, (uint32_t)(seed >> 32), mask_b);
        else if constexpr (POW2)
          off = row_off_u32<SH>(klo[u], klo[u] >> 30, hh.c0, hh.c2, mask_b);
        else
          off = (uint32_t)fmod64(mix64(((uint64_t)khi[u] << 32 | klo[u]) ^ seed), wm) << SH;
        c[4 * j + u] = *reinterpret_cast<const CT*>(rowb + off);
      }
    }
    if (it >= NB) mbar_wait(empty_a + 8 * pb, (uint32_t)((it >> LNB) - 1) & 1);
#pragma unroll
    for (int j = 0; j < KPL / 4; ++j) {
      const uint32_t dst = o_recv[j] + pb * RB;
      if constexpr (U16)
        st_async_v2(dst, c[4 * j] | (c[4 * j + 1] << 16), c[4 * j + 2] | (c[4 * j + 3] << 16), o_full[j] + 8 * pb);
      else
        st_async_v4(dst, c[4 * j], c[4 * j + 1], c[4 * j + 2], c[4 * j + 3], o_full[j] + 8 * pb);
    }

    if (it >= 1) owner_phase(it - 1, (it - 1) & (NB - 1), (uint32_t)((it - 1) >> LNB) & 1, tile_key - tstep);
    tile_key += tstep;
  }
  if (Tw > 0) owner_phase(Tw - 1, (Tw - 1) & (NB - 1), (uint32_t)((Tw - 1) >> LNB) & 1, tile_key - tstep);
  cluster_sync_all();  // no CTA exits while peers may still touch its shared memory
}




// Launch the warp-pipelined cluster kernel for u32 / u64 keys (16-B aligned
// keys and output); the < K-key tail goes to the L2 kernel. Returns -1 if not
// suited.
template <int D, typename CT, bool POW2, bool KU64>
static int try_cw_k(const uint32_t* counters, const Seeds<D>& sd, Mod wm, int64_t w, KeySrc ks, int64_t n,
                    int64_t* out, cudaStream_t st, int optin) {
  constexpr int NW = SFK_CW_NW, NB = SFK_CW_NB;
  // owner phase: KPL / D keys per lane; u64 keys take half the tile of u32
  // ones at d = 4 (the prefetched keys' registers)
  constexpr int KPL = D == 2 ? 8 : D == 8 ? 16 : (KU64 ? 8 : SFK_CW_KPL);
  constexpr int K = 32 * KPL;
  if ((reinterpret_cast<uintptr_t>(ks.p) & 15) || (reinterpret_cast<uintptr_t>(out) & 15)) return -1;
  const int64_t ntiles = n / K;
  if (ntiles < 1) return -1;
  const size_t row_bytes = ((size_t)w * sizeof(CT) + 15) & ~size_t(15);
  const size_t smem = row_bytes + (sizeof(CT) == 2 ? 2 * OVF_STRIDE * 4 : 0) + (size_t)NW * NB * K * sizeof(CT) +
                      (size_t)NW * 2 * NB * 8;
  if (smem > (size_t)optin) return -1;
  if (sizeof(CT) == 2 && (size_t)NW * NB * K * sizeof(CT) < (size_t)OVF_SLOTS * 4) return -1;  // setup scratch
  auto kern = min_query_cw<D, CT, NW, KPL, NB, POW2, KU64>;
  // the opt-in attribute belongs to the current device's context: set it per call
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = D;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.blockDim = dim3(NW * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.gridDim = dim3(D * sm_count());
  int nclusters = 0;
  if (cudaOccupancyMaxActiveClusters(&nclusters, kern, &cfg) != cudaSuccess || nclusters <= 0) {
    cudaGetLastError();
    return -1;
  }
  const int64_t need = (ntiles + NW - 1) / NW;
  if ((int64_t)nclusters > need) nclusters = (int)need;
  cfg.gridDim = dim3(D * nclusters);
  note_launch();
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, counters, sd, wm, w, ks.p, ntiles, out);
  if (e != cudaSuccess) {
    set_error("min_query_cw launch: %s", cudaGetErrorString(e));
    return (int)e;
  }
  int rc = check_launch("min_query_cw");
  if (rc) return rc;
  g_query_last = 4;
  const int64_t done = ntiles * K;
  if (done < n) {
    KeySrc tail{static_cast<const char*>(ks.p) + done * (KU64 ? 8 : 4), ks.kind, 0};
    note_launch();
    min_query_l2<D, 4><<<grid_for(n - done, 256 * 4, sm_count() * 8), 256, 0, st>>>(counters, sd, wm, w, tail,
                                                                                    n - done, out + done);
    rc = check_launch("min_query_l2 (tail)");
  }
  return rc;
}

template <int D, typename CT, bool POW2>
static int try_cw(const uint32_t* counters, const Seeds<D>& sd, Mod wm, int64_t w, KeySrc ks, int64_t n,
                  int64_t* out, cudaStream_t st, int optin) {
  if (ks.kind == SFK_KEY_U32) return try_cw_k<D, CT, POW2, false>(counters, sd, wm, w, ks, n, out, st, optin);
  if (ks.kind == SFK_KEY_U64) return try_cw_k<D, CT, POW2, true>(counters, sd, wm, w, ks, n, out, st, optin);
  return -1;
}

// Launch the cluster kernel if this (d, w, n) suits it; returns -1 if not.
template <int D, typename CT, int TILE, int KK, bool VEC, bool POW2>
static int try_cluster_k(const uint32_t* counters, const Seeds<D>& sd, Mod wm, int64_t w, KeySrc ks, int64_t n,
                         int64_t* out, cudaStream_t st, int optin) {
  constexpr int NT = SFK_QUERY_NT;
  constexpr int Q = ((TILE + D - 1) / D + 3) & ~3;
  const size_t row_bytes = ((size_t)w * sizeof(CT) + 15) & ~size_t(15);
  const size_t smem = row_bytes + (sizeof(CT) == 2 ? 2 * OVF_STRIDE * 4 : 0) + (size_t)QNB * D * Q * sizeof(CT) +
                      2 * QNB * 8;
  if (smem + 1024 > (size_t)optin) return -1;
  auto kern = min_query_cluster<D, CT, TILE, NT, KK, VEC, POW2>;
  // the opt-in attribute belongs to the current device's context: set it per call
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 1024) != cudaSuccess) {
    cudaGetLastError();
    return -1;
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
  const int out_vec = (reinterpret_cast<uintptr_t>(out) & 15) == 0;
  note_launch();
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, counters, sd, wm, w, ks, n, out, out_vec);
  if (e != cudaSuccess) {
    set_error("min_query_cluster launch: %s", cudaGetErrorString(e));
    return (int)e;
  }
  g_query_last = 3;
  return check_launch("min_query_cluster");
}

template <int D, typename CT, int TILE, bool POW2>
static int try_cluster_p(const uint32_t* counters, const Seeds<D>& sd, Mod wm, int64_t w, KeySrc ks, int64_t n,
                         int64_t* out, cudaStream_t st, int optin) {
  if (ks.kind == SFK_KEY_U32) {
    // 512 threads x 16 keys each per tile measured faster than 1024 x 8
    if ((reinterpret_cast<uintptr_t>(ks.p) & 15) == 0)
      return try_cluster_k<D, CT, TILE, SFK_KEY_U32, true, POW2>(counters, sd, wm, w, ks, n, out, st, optin);
    return try_cluster_k<D, CT, TILE, SFK_KEY_U32, false, POW2>(counters, sd, wm, w, ks, n, out, st, optin);
  }
  if (ks.kind == SFK_KEY_U64)
    return try_cluster_k<D, CT, TILE, SFK_KEY_U64, false, POW2>(counters, sd, wm, w, ks, n, out, st, optin);
  return try_cluster_k<D, CT, TILE, SFK_KEY_RECORD, false, POW2>(counters, sd, wm, w, ks, n, out, st, optin);
}

template <int D, typename CT, int TILE>
static int try_cluster(const uint32_t* counters, const Seeds<D>& sd, Mod wm, int64_t w, KeySrc ks, int64_t n,
                       int64_t* out, cudaStream_t st, int optin) {
  if (wm.pow2 && w <= (int64_t(1) << 32))
    return try_cluster_p<D, CT, TILE, true>(counters, sd, wm, w, ks, n, out, st, optin);
  return try_cluster_p<D, CT, TILE, false>(counters, sd, wm, w, ks, n, out, st, optin);
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
  const int optin = smem_optin();
  const size_t tab_bytes = (size_t)D * (size_t)w * 4;
  const int mode = g_query_path;
  // staging costs tab_bytes per SM; worth it once the batch's own gathers
  // dwarf it (>= ~16 keys per staged counter word across the chip)
  const bool smem_fits = tab_bytes <= (size_t)optin;
  const bool smem_pays = (double)n * D >= 16.0 * (double)sms * (double)(D * w) / 4.0;
  if ((mode == 0 && smem_fits && smem_pays) || (mode == 2 && smem_fits)) {
    if (cudaFuncSetAttribute(min_query_smem<D, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin) != cudaSuccess) {
      set_error("min_query_smem: cudaFuncSetAttribute: %s", cudaGetErrorString(cudaGetLastError()));
      return 1;
    }
    { note_launch(); min_query_smem<D, 4><<<sms, 1024, tab_bytes, st>>>(counters, sd, wm, w, ks, n, out); }
    g_query_last = 2;
    return check_launch("min_query_smem");
  }
  // row-partitioned cluster path: d CTAs per cluster (portable size <= 8);
  // pays once the batch is well beyond the per-CTA row staging (~2M keys)
  // warp-pipelined cluster path (u32 keys, d in {2, 4, 8}): u32 rows when
  // they fit beside the rings, else u16 codes
  if constexpr (D == 2 || D == 4 || D == 8) {
    if ((mode == 0 && !smem_fits && n >= (int64_t(1) << 21)) || mode == 4) {
      int rc = -1;
      if ((size_t)w * 4 + 100 * 1024 <= (size_t)optin) {
        rc = wm.pow2 ? try_cw<D, uint32_t, true>(counters, sd, wm, w, ks, n, out, st, optin)
                     : try_cw<D, uint32_t, false>(counters, sd, wm, w, ks, n, out, st, optin);
      }
      if (rc < 0 && w <= 65536)
        rc = wm.pow2 ? try_cw<D, uint16_t, true>(counters, sd, wm, w, ks, n, out, st, optin)
                     : try_cw<D, uint16_t, false>(counters, sd, wm, w, ks, n, out, st, optin);
      if (rc >= 0) return rc;
    }
  }
  if (D >= 2 && D <= 8 && ((mode == 0 && !smem_fits && n >= (int64_t(1) << 21)) || mode == 3 || mode == 4)) {
    int rc = -1;
    if ((size_t)w * 4 + 2 * 8192 * 4 + 64 + 1024 <= (size_t)optin)
      rc = try_cluster<D, uint32_t, 8192>(counters, sd, wm, w, ks, n, out, st, optin);
    else
      rc = try_cluster<D, uint16_t, SFK_QUERY_TILE>(counters, sd, wm, w, ks, n, out, st, optin);
    if (rc >= 0) return rc;
  }
  int blocks = grid_for(n, 256 * 4, sms * 8);
  { note_launch(); min_query_l2<D, 4><<<blocks, 256, 0, st>>>(counters, sd, wm, w, ks, n, out); }
  g_query_last = 1;
  return check_launch("min_query_l2");
}


// ---- two-phase query: row indices now, gathers later ------------------------
// sfk_query_index writes, for each key t and row r, its bucket index as u16
// at idx[r * n + t] (needs w <= 65536). sfk_min_query_idx then gathers and
// takes the min from those indices; the cluster kernel runs with
// KK = KEY_IDX16 and reads 2 B per key and row instead of hashing. The index
// pass reads 4 B and writes 2d B per key; it does not need the counters, so
// it can run while the sketch is still being built.
template <int D>
__global__ void __launch_bounds__(256) query_index_k(Seeds<D> seeds, Mod wm, KeySrc keys, int64_t n,
                                                     uint16_t* __restrict__ idx, int vec_ok) {
  U32Hash h[D];
#pragma unroll
  for (int i = 0; i < D; ++i) h[i] = make_u32hash(seeds.s[i]);
  const uint32_t mask = (uint32_t)wm.mask;
  const bool fast = vec_ok && keys.kind == SFK_KEY_U32 && wm.pow2;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 4;
  for (int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; t < n; t += stride) {
    if (fast && t + 3 < n) {
      const uint4 k = __ldcs(reinterpret_cast<const uint4*>(static_cast<const uint32_t*>(keys.p) + t));
#pragma unroll
      for (int i = 0; i < D; ++i) {
        const uint32_t a0 = row_index_u32(k.x, h[i], mask), a1 = row_index_u32(k.y, h[i], mask);
        const uint32_t a2 = row_index_u32(k.z, h[i], mask), a3 = row_index_u32(k.w, h[i], mask);
        __stcs(reinterpret_cast<uint2*>(idx + (int64_t)i * n + t), make_uint2(a0 | (a1 << 16), a2 | (a3 << 16)));
      }
    } else {
      for (int u = 0; u < 4 && t + u < n; ++u) {
        const uint64_t key = load_key(keys, t + u);
#pragma unroll
        for (int i = 0; i < D; ++i) idx[(int64_t)i * n + t + u] = (uint16_t)fmod64(mix64(key ^ seeds.s[i]), wm);
      }
    }
  }
}

template <int D>
__global__ void __launch_bounds__(256) min_query_idx_l2(const uint32_t* __restrict__ counters, int64_t w,
                                                        const uint16_t* __restrict__ idx, int64_t n,
                                                        int64_t* __restrict__ out) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    uint32_t m = U32MAX;
#pragma unroll
    for (int i = 0; i < D; ++i) m = min(m, __ldg(counters + (int64_t)i * w + idx[(int64_t)i * n + t]));
    out[t] = (int64_t)m;
  }
}

template <int D>
static int launch_index_d(const uint64_t* seeds_host, int64_t w, KeySrc ks, int64_t n, uint16_t* idx, cudaStream_t st) {
  Seeds<D> sd;
  for (int i = 0; i < D; ++i) sd.s[i] = seeds_host[i];
  const int vec_ok = ks.kind == SFK_KEY_U32 && (reinterpret_cast<uintptr_t>(ks.p) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(idx) & 7) == 0 && (n & 3) == 0;
  { note_launch(); query_index_k<D><<<grid_for((n + 3) / 4, 256, sm_count() * 8), 256, 0, st>>>(sd, make_mod((uint64_t)w), ks, n, idx, vec_ok); }
  return check_launch("query_index");
}

template <int D>
static int launch_query_idx_d(const uint32_t* counters, int64_t w, const uint16_t* idx, int64_t n, int64_t* out,
                              cudaStream_t st) {
  const int optin = smem_optin();
  Seeds<D> sd{};
  const Mod wm = make_mod((uint64_t)w);
  const KeySrc ks{idx, KEY_IDX16, 0};
  const bool vec = (reinterpret_cast<uintptr_t>(idx) & 7) == 0 && (n & 3) == 0;
  if (D >= 2 && D <= 8 && g_query_path != 1 && n >= (int64_t(1) << 21)) {
    int rc = vec ? try_cluster_k<D, uint16_t, 8192, KEY_IDX16, true, true>(counters, sd, wm, w, ks, n, out, st, optin)
                 : try_cluster_k<D, uint16_t, 8192, KEY_IDX16, false, true>(counters, sd, wm, w, ks, n, out, st, optin);
    if (rc >= 0) return rc;
  }
  { note_launch(); min_query_idx_l2<D><<<grid_for(n, 256, sm_count() * 8), 256, 0, st>>>(counters, w, idx, n, out); }
  g_query_last = 1;
  return check_launch("min_query_idx_l2");
}

int launch_query_index(const uint64_t* seeds_host, int d, int64_t w, KeySrc ks, int64_t n, uint16_t* idx,
                       cudaStream_t st) {
  if (n <= 0) return 0;
  if (w > 65536) {
    set_error("sfk_query_index: w=%lld exceeds the u16 index range", (long long)w);
    return 1;
  }
  switch (d) {
    case 1: return launch_index_d<1>(seeds_host, w, ks, n, idx, st);
    case 2: return launch_index_d<2>(seeds_host, w, ks, n, idx, st);
    case 3: return launch_index_d<3>(seeds_host, w, ks, n, idx, st);
    case 4: return launch_index_d<4>(seeds_host, w, ks, n, idx, st);
    case 5: return launch_index_d<5>(seeds_host, w, ks, n, idx, st);
    case 6: return launch_index_d<6>(seeds_host, w, ks, n, idx, st);
    case 7: return launch_index_d<7>(seeds_host, w, ks, n, idx, st);
    case 8: return launch_index_d<8>(seeds_host, w, ks, n, idx, st);
  }
  set_error("sfk_query_index: unsupported d=%d", d);
  return 1;
}

int launch_min_query_idx(const uint32_t* counters, int d, int64_t w, const uint16_t* idx, int64_t n, int64_t* out,
                         cudaStream_t st) {
  if (n <= 0) return 0;
  if (w > 65536) {
    set_error("sfk_min_query_idx: w=%lld exceeds the u16 index range", (long long)w);
    return 1;
  }
  switch (d) {
    case 1: return launch_query_idx_d<1>(counters, w, idx, n, out, st);
    case 2: return launch_query_idx_d<2>(counters, w, idx, n, out, st);
    case 3: return launch_query_idx_d<3>(counters, w, idx, n, out, st);
    case 4: return launch_query_idx_d<4>(counters, w, idx, n, out, st);
    case 5: return launch_query_idx_d<5>(counters, w, idx, n, out, st);
    case 6: return launch_query_idx_d<6>(counters, w, idx, n, out, st);
    case 7: return launch_query_idx_d<7>(counters, w, idx, n, out, st);
    case 8: return launch_query_idx_d<8>(counters, w, idx, n, out, st);
  }
  set_error("sfk_min_query_idx: unsupported d=%d", d);
  return 1;
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
