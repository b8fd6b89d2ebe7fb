// Latency floor of the ordered engine's dependency hop.
//
// A hop of the engine is: a run publishes its slim cells with relaxed
// gpu-scope stores, and the run waiting on them observes the new sequence
// number with relaxed gpu-scope loads (polling). This measures that hand-off
// in isolation: two CTAs on different SMs ping-pong a counter R times; one
// hop = half a round trip. Also measured: the same ping-pong while every other SM
// runs 8 warps that poll random cells of a 2 MiB table (the engine's
// background load). The engine's critical path x the idle hop latency is its
// latency roofline. Round 2 adds hot-spot backgrounds: the pollers hit only
// `hot` distinct cells (1 = the ping-pong cell itself, 64 = a few hot cells
// elsewhere), as lanes waiting on the same hot slim cells do.
//
// Output: one JSON object on stdout.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hop_latency hop_latency.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ unsigned long long ld_rel(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// blocks 0 and 1: the ping-pong pair (thread 0 each); other blocks: pollers
__global__ void pingpong(unsigned long long* cell, int rounds, unsigned long long* ns_out,
                         unsigned long long* table, uint32_t mask, volatile int* stop, int hot) {
  if (blockIdx.x >= 2) {  // background load: random relaxed polls
    uint32_t s = 0x9E3779B9u * (blockIdx.x * blockDim.x + threadIdx.x + 1);
    unsigned long long acc = 0;
    while (!*stop) {
#pragma unroll 4
      for (int i = 0; i < 64; ++i) {
        s ^= s << 13; s ^= s >> 17; s ^= s << 5;
        const unsigned long long* p = hot == 1 ? cell : hot > 1 ? table + (s % hot) * 4096 : table + (s & mask);
        acc += ld_rel(p);
      }
    }
    if (acc == 42) table[0] = acc;
    return;
  }
  if (threadIdx.x != 0) return;
  const int me = blockIdx.x;  // 0 starts
  unsigned long long t0 = gtimer();
  for (int r = 0; r < rounds; ++r) {
    const unsigned long long want = 2ull * r + me;
    while (ld_rel(cell) != want) {
    }
    st_rel(cell, want + 1);
  }
  if (me == 0) {
    ns_out[0] = gtimer() - t0;
    *stop = 1;
  }
}

int main() {
  const int rounds = 20000;
  unsigned long long *cell, *ns, *table;
  int* stop;
  const size_t tab_words = (2u << 20) / 8;  // 2 MiB: the packed cfg-3 slim
  CK(cudaMalloc(&cell, 256));
  CK(cudaMalloc(&ns, 8));
  CK(cudaMalloc(&table, tab_words * 8));
  CK(cudaMalloc(&stop, 4));
  CK(cudaMemset(table, 0, tab_words * 8));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double res[4];
  const int hots[4] = {0, 0, 1, 64};
  for (int loaded = 0; loaded < 4; ++loaded) {
    double best = 1e30;
    for (int rep = 0; rep < 3; ++rep) {
      CK(cudaMemset(cell, 0, 256));
      CK(cudaMemset(stop, 0, 4));
      const int blocks = loaded ? sms : 2;
      pingpong<<<blocks, loaded ? 256 : 32>>>(cell, rounds, ns, table, (uint32_t)(tab_words - 1), stop, hots[loaded]);
      CK(cudaGetLastError());
      CK(cudaDeviceSynchronize());
      unsigned long long h = 0;
      CK(cudaMemcpy(&h, ns, 8, cudaMemcpyDeviceToHost));
      const double hop = (double)h / (2.0 * rounds);
      if (hop < best) best = hop;
    }
    res[loaded] = best;
  }
  printf("{\"hop_ns_idle\": %.1f, \"hop_ns_loaded\": %.1f, \"hop_ns_hot_same_cell\": %.1f, "
         "\"hop_ns_hot_64_cells\": %.1f, \"rounds\": %d, \"background\": "
         "\"%d CTAs x 256 threads polling a 2 MiB table / the ping-pong cell / 64 hot cells\"}\n",
         res[0], res[1], res[2], res[3], rounds, sms - 2);
  return 0;
}
