// Microbenchmark of the SFF run replay (one lane, one long synthetic run).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/replay_bench tools/replay_bench.cu
#include "../paper_1701_04148_b200/csrc/sfk_sf.cu"

#include <cstdio>
#include <vector>
#include <random>

namespace sfk {
void note_launch() {}
void set_error(const char*, ...) {}
int check_launch(const char*) { return 0; }
int sm_count() { return 148; }
}  // namespace sfk

using namespace sfk;

__global__ void bench_k(EngineArgs<4> a, uint32_t L, uint32_t bits0, uint32_t A0v, uint32_t W1, uint32_t W2,
                        uint32_t W3, unsigned long long* out) {
  __shared__ uint32_t lut[256];
  __shared__ uint8_t rlut[WMAX * 8 * 256];
  build_step_lut(lut);
  build_reflect_lut(rlut);
  __syncthreads();
  if (threadIdx.x != 0) return;
  uint32_t A[4] = {A0v, A0v + W1, A0v + W2, A0v + W3}, O[4] = {5, 5, 5, 5};
  uint32_t c[4] = {A0v, A0v, A0v + 1, A0v}, raised[4] = {0, 0, 0, 0}, ws[3] = {0, 0, 0};
  Cursor k{};
  k.m = A0v;
  k.A0 = A0v;
  k.x = 0;
  k.e = 0;
  k.rem = L;
  k.ring = false;
  const long long t0 = clock64();
  while (!replay_step<4, 2>(a, k, 0u, L | 0x80000000u, bits0, A, O, c, raised, ws, lut, rlut)) {
  }
  const long long t1 = clock64();
  out[0] = t1 - t0;
  out[1] = ws[0];
  out[2] = ws[1];
  out[3] = ws[2];
  out[4] = c[0] + c[1] + c[2] + c[3] + raised[0] + raised[1] + raised[2] + raised[3];
}

int main(int argc, char** argv) {
  const uint32_t L = 1u << 20;
  const double pdel = argc > 1 ? atof(argv[1]) : 0.2;
  std::mt19937 g(1);
  std::bernoulli_distribution bd(pdel);
  std::vector<uint32_t> bits(L / 32 + 16, 0);
  for (uint32_t e = 0; e < L; ++e)
    if (bd(g)) bits[e >> 5] |= 1u << (e & 31);
  uint32_t* d_bits;
  cudaMalloc(&d_bits, bits.size() * 4);
  cudaMemcpy(d_bits, bits.data(), bits.size() * 4, cudaMemcpyHostToDevice);
  unsigned long long* d_out;
  cudaMalloc(&d_out, 64);
  EngineArgs<4> a{};
  std::vector<uint32_t> hw(bits.size());
  a.delbits = d_bits;
  uint32_t* d_ws;
  cudaMalloc(&d_ws, bits.size() * 4 + 256);
  word_sums_k<<<64, 256>>>(d_bits, (uint32_t)bits.size(), d_ws);
  a.wsum = d_ws;
  a.budget = 0xFFFFFFFFu;
  const uint32_t Ws[][3] = {{0, 0, 0}, {2, 3, 5}, {20, 30, 50}};
  for (auto& w : Ws) {
    for (int rep = 0; rep < 2; ++rep) {
      bench_k<<<1, 256>>>(a, L, bits[0], 1000000, w[0], w[1], w[2], d_out);
      unsigned long long h[5];
      cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
      if (rep)
        printf("pdel=%.2f W={%u,%u,%u}: %.1f cycles/op (gap %llu steady %llu slow %llu words)\n", pdel, w[0], w[1], w[2],
               (double)h[0] / L, h[1], h[2], h[3]);
    }
  }
  return 0;
}
