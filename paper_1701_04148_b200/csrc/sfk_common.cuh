// Shared device primitives for the SF sketch kernels: the reference's hash
// family (hashing.py:33-45, _kernels.py:44-53), exact 64-bit range
// reduction, key loading for the three key kinds, and error plumbing.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstddef>

#include "../../include/sfsketch_cuda.h"

namespace sfk {

constexpr uint32_t U32MAX = 0xFFFFFFFFu;
constexpr uint64_t U64MAX = 0xFFFFFFFFFFFFFFFFull;
constexpr uint32_t NONE32 = 0xFFFFFFFFu;
constexpr int MAXD = 8;       // rows handled by the templated parallel kernels
constexpr int MAXSEEDS = 64;  // rows accepted at all (seeds travel by value)

// finalize64 (hashing.py:33-45) == _mix (_kernels.py:44-48). Wrapping u64.
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// Exact unsigned 64-bit x % m (the reference's `% modulus`, _kernels.py:53).
// Power-of-two ranges use a mask. Otherwise q = umulhi(x, floor((2^64-1)/m))
// satisfies q <= x/m < q + 2, so at most two corrections give the exact
// remainder for every x.
struct Mod {
  uint64_t m;
  uint64_t magic;
  uint64_t mask;
  int pow2;
};

inline Mod make_mod(uint64_t m) {
  Mod r;
  r.m = m;
  r.pow2 = (m & (m - 1)) == 0;
  r.mask = m - 1;
  r.magic = m ? (0xFFFFFFFFFFFFFFFFull / m) : 0;
  return r;
}

__device__ __forceinline__ uint64_t fmod64(uint64_t x, const Mod& M) {
  if (M.pow2) return x & M.mask;
  uint64_t q = __umul64hi(x, M.magic);
  uint64_t r = x - q * M.m;
  if (r >= M.m) r -= M.m;
  if (r >= M.m) r -= M.m;
  return r;
}

// _bucket (_kernels.py:51-53)
__device__ __forceinline__ uint64_t bucket(uint64_t key, uint64_t seed, const Mod& M) {
  return fmod64(mix64(key ^ seed), M);
}

struct KeySrc {
  const void* p;
  int kind;
  int rec;
};

// FNV-1a-64 over `rec` bytes then finalize64 (hashing.py:124-129).
__device__ __forceinline__ uint64_t record_key(const uint8_t* r, int rec) {
  uint64_t h = 0xCBF29CE484222325ull;
  for (int b = 0; b < rec; ++b) h = (h ^ (uint64_t)r[b]) * 0x100000001B3ull;
  return mix64(h);
}

__device__ __forceinline__ uint64_t load_key(const KeySrc& k, int64_t t) {
  if (k.kind == SFK_KEY_U64) return __ldg(static_cast<const unsigned long long*>(k.p) + t);
  if (k.kind == SFK_KEY_U32) return (uint64_t)__ldg(static_cast<const unsigned int*>(k.p) + t);
  return record_key(static_cast<const uint8_t*>(k.p) + t * (int64_t)k.rec, k.rec);
}

template <int N>
struct Seeds {
  uint64_t s[N];
};

// Relaxed gpu-scope 64-bit load/store: coherent at L2, never served from a
// stale L1 line. Used for the packed (seq << 32 | value) slim cells of the
// ordered engine.
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Workspace carving: 256-B aligned sub-allocations from one caller buffer.
struct Carver {
  char* base;
  size_t off;
  size_t cap;
  bool ok;
  explicit Carver(void* b, size_t c) : base(static_cast<char*>(b)), off(0), cap(c), ok(true) {}
  template <typename T>
  T* take(size_t count) {
    size_t bytes = (count * sizeof(T) + 255) & ~size_t(255);
    T* p = reinterpret_cast<T*>(base ? base + off : nullptr);
    off += bytes;
    if (off > cap) ok = false;
    return p;
  }
};

// ops/counters statistics for the CM/CU prechecks
struct Stats {
  unsigned long long n_ins, n_del;
  unsigned long long first_del;  // min index of a delete (or n)
  unsigned long long ins_before_first_del;
  uint32_t cmax, cmin;
  unsigned long long first_bad;  // min index of an op code other than 0 / 1 (or n)
};

// per-op gate inputs of the gated engine kinds (sfk_sf.cu kinds 7 and 8)
struct ExtArgs {
  uint16_t* exps;              // CML exponents (d, w)
  const double* gate;          // CML: gate[c] = base ** -c, 65536 entries, non-increasing
  uint64_t rng_seed;           // CML coin-flip stream seed
  int64_t start_pos;           // CML: inserts before this chunk
  const int64_t* true_counts;  // oracle-assisted: exact post-insert counts
};

// counts every kernel this library launches itself (CUB's internal sort/scan
// launches are not included); read through sfk_launch_count()
void note_launch();

void set_error(const char* fmt, ...);
int check_launch(const char* where);

inline int grid_for(int64_t n, int threads, int cap_blocks) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > cap_blocks) b = cap_blocks;
  return (int)b;
}

int sm_count();

}  // namespace sfk
