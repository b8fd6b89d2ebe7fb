// Roofline denominators for the SF sketch hot path.
//
// Measures, on the B200 this runs on, the peak rate of the memory operations
// the sketch kernels are built from:
//   * random 4-B gathers from shared memory (bank conflicts included),
//   * random 4-B gathers from tables of 256 KiB / 1 MiB / 4 MiB / 64 MiB
//     (L2-resident) and 1 GiB (HBM),
//   * random 4-B atomicAdd (no return, RED) and with return (ATOM) into
//     1 MiB / 4 MiB / 64 MiB tables,
//   * streaming copy bandwidth.
// Each figure is the best of several CUDA-event-timed launches after warm-up.
// Output: one JSON object on stdout (written to profiles/ by the caller).
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_peaks gather_peaks.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint32_t xs32(uint32_t x) { x ^= x << 13; x ^= x >> 17; x ^= x << 5; return x; }

// Every thread performs ITER random 4-B loads, 4 independent streams for MLP.
template <int ITER>
__global__ void gather_global(const uint32_t* __restrict__ tab, uint32_t mask, uint32_t* out) {
  uint32_t s0 = 0x9E3779B9u * (blockIdx.x * blockDim.x + threadIdx.x + 1);
  uint32_t s1 = xs32(s0 ^ 0x1234567u), s2 = xs32(s1 ^ 0x89abcdefu), s3 = xs32(s2 ^ 0x5555u);
  uint32_t acc = 0;
#pragma unroll 4
  for (int it = 0; it < ITER; it += 4) {
    s0 = xs32(s0); s1 = xs32(s1); s2 = xs32(s2); s3 = xs32(s3);
    acc += __ldg(tab + (s0 & mask)) ^ __ldg(tab + (s1 & mask)) ^ __ldg(tab + (s2 & mask)) ^ __ldg(tab + (s3 & mask));
  }
  if (acc == 0x7fffffffu) out[0] = acc;
}

template <int ITER>
__global__ void gather_smem(const uint32_t* __restrict__ tab, uint32_t words, uint32_t* out) {
  extern __shared__ uint32_t sm[];
  for (uint32_t k = threadIdx.x; k < words; k += blockDim.x) sm[k] = tab[k];
  __syncthreads();
  uint32_t mask = words - 1;
  uint32_t s0 = 0x9E3779B9u * (blockIdx.x * blockDim.x + threadIdx.x + 1);
  uint32_t s1 = xs32(s0 ^ 0x1234567u), s2 = xs32(s1 ^ 0x89abcdefu), s3 = xs32(s2 ^ 0x5555u);
  uint32_t acc = 0;
#pragma unroll 4
  for (int it = 0; it < ITER; it += 4) {
    s0 = xs32(s0); s1 = xs32(s1); s2 = xs32(s2); s3 = xs32(s3);
    acc += sm[s0 & mask] ^ sm[s1 & mask] ^ sm[s2 & mask] ^ sm[s3 & mask];
  }
  if (acc == 0x7fffffffu) out[0] = acc;
}

template <int ITER, bool RET>
__global__ void atomic_rand(uint32_t* tab, uint32_t mask, uint32_t* out) {
  uint32_t s0 = 0x9E3779B9u * (blockIdx.x * blockDim.x + threadIdx.x + 1);
  uint32_t acc = 0;
#pragma unroll 4
  for (int it = 0; it < ITER; ++it) {
    s0 = xs32(s0);
    if (RET) acc += atomicAdd(tab + (s0 & mask), 1u);
    else atomicAdd(tab + (s0 & mask), 1u);
  }
  if (RET && acc == 0x7fffffffu) out[0] = acc;
}

__global__ void copy_k(const uint4* __restrict__ a, uint4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

template <typename F>
static float best_ms(F f, int reps = 7) {
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  f(); f(); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(a)); f(); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
    float ms; CK(cudaEventElapsedTime(&ms, a, b)); best = std::min(best, ms);
  }
  CK(cudaGetLastError());
  return best;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int optin = 0; CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0));
  int sms = p.multiProcessorCount;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"smem_optin\": %d, \"clock_khz\": %d", p.name, sms, p.l2CacheSize, optin, p.clockRate);
  uint32_t* out; CK(cudaMalloc(&out, 64));
  const size_t big = 1ull << 28;  // 1 GiB of u32
  uint32_t* tab; CK(cudaMalloc(&tab, big * 4)); CK(cudaMemset(tab, 1, big * 4));
  constexpr int IT = 256;
  const int threads = 512, blocks = sms * 4;
  const double nload = (double)blocks * threads * IT;
  // global gathers
  size_t sizes[] = {1u << 16, 1u << 18, 1u << 20, 1u << 24, 1u << 28};
  const char* names[] = {"256KiB", "1MiB", "4MiB", "64MiB", "1GiB"};
  for (int s = 0; s < 5; ++s) {
    uint32_t mask = (uint32_t)(sizes[s] - 1);
    float ms = best_ms([&] { gather_global<IT><<<blocks, threads>>>(tab, mask, out); });
    printf(", \"gather_%s_Gps\": %.2f", names[s], nload / ms / 1e6);
  }
  // smem gathers: 128 KiB table (power of two that fits)
  {
    uint32_t words = 1u << 15;
    CK(cudaFuncSetAttribute(gather_smem<IT * 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, words * 4));
    float ms = best_ms([&] { gather_smem<IT * 4><<<sms, 1024, words * 4>>>(tab, words, out); });
    double n = (double)sms * 1024 * IT * 4;
    printf(", \"gather_smem128KiB_Gps\": %.2f", n / ms / 1e6);
  }
  // atomics
  size_t asizes[] = {1u << 18, 1u << 20, 1u << 24};
  const char* anames[] = {"1MiB", "4MiB", "64MiB"};
  constexpr int AIT = 64;
  const double natom = (double)blocks * threads * AIT;
  for (int s = 0; s < 3; ++s) {
    uint32_t mask = (uint32_t)(asizes[s] - 1);
    float ms = best_ms([&] { atomic_rand<AIT, false><<<blocks, threads>>>(tab, mask, out); });
    printf(", \"red_%s_Gps\": %.2f", anames[s], natom / ms / 1e6);
    ms = best_ms([&] { atomic_rand<AIT, true><<<blocks, threads>>>(tab, mask, out); });
    printf(", \"atom_ret_%s_Gps\": %.2f", anames[s], natom / ms / 1e6);
  }
  // copy
  {
    size_t n16 = big * 4 / 2 / 16;
    uint4* a = (uint4*)tab; uint4* b = a + n16;
    float ms = best_ms([&] { copy_k<<<sms * 8, 512>>>(a, b, n16); });
    printf(", \"copy_GBps\": %.1f", 2.0 * n16 * 16 / ms / 1e6);
  }
  printf("}\n");
  return 0;
}
