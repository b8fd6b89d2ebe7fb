// Host <-> device I/O probe for the e2e query path (DESIGN.md §5 e2e):
// pinned H2D / D2H rates alone and concurrently, and how fast host threads
// can widen 2-B / 4-B per-query results into the int64 output the API
// returns. Prints one JSON object per line.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -Xcompiler -mavx512f,-mavx512bw,-fopenmp \
//        tools/host_io_probe.cu -o tools/host_io_probe
#include <cuda_runtime.h>
#include <immintrin.h>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

// copy `bytes` in `chunk`-byte pieces round-robin over `ns` streams
static void copies(void* dst, const void* src, size_t bytes, size_t chunk, cudaMemcpyKind k, cudaStream_t* s, int ns) {
    size_t c = 0;
    for (size_t a = 0; a < bytes; a += chunk, ++c) {
        size_t b = bytes - a < chunk ? bytes - a : chunk;
        cudaMemcpyAsync((char*)dst + a, (const char*)src + a, b, k, s[c % ns]);
    }
}

template <class F>
static double par(int T, F f) {
    std::vector<std::thread> th;
    double t0 = now();
    for (int i = 0; i < T; ++i) th.emplace_back(f, i, T);
    for (auto& t : th) t.join();
    return now() - t0;
}

int main(int argc, char** argv) {
    size_t n = argc > 1 ? strtoull(argv[1], 0, 10) : (1ull << 29);  // queries
    int hw = (int)std::thread::hardware_concurrency();
    printf("{\"probe\": \"cpu\", \"hardware_concurrency\": %d, \"n\": %zu}\n", hw, n);
    uint32_t *hk, *hc32;
    uint16_t* hc16;
    int64_t* ho;
    CK(cudaHostAlloc(&hk, n * 4, 0));
    CK(cudaHostAlloc(&hc32, n * 4, 0));
    CK(cudaHostAlloc(&hc16, n * 2, 0));
    CK(cudaHostAlloc(&ho, n * 8, 0));
    void *dk, *do_;
    CK(cudaMalloc(&dk, n * 4));
    CK(cudaMalloc(&do_, n * 8));
    memset(hk, 1, n * 4);
    memset(hc32, 0, n * 4);
    memset(hc16, 0, n * 2);
    memset(ho, 0, n * 8);
    for (size_t i = 0; i < n; ++i) hc16[i] = (uint16_t)(i * 2654435761u >> 16);
    cudaStream_t s[4];
    for (auto& x : s) CK(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
    const size_t chunk = 1 << 25;
    auto run = [&](const char* name, size_t h2d, size_t d2h) {
        for (int rep = 0; rep < 3; ++rep) {
            CK(cudaDeviceSynchronize());
            double t0 = now();
            if (h2d) copies(dk, hk, h2d, chunk, cudaMemcpyHostToDevice, s, 2);
            if (d2h) copies(ho, do_, d2h, chunk, cudaMemcpyDeviceToHost, s + 2, 2);
            CK(cudaDeviceSynchronize());
            double t = now() - t0;
            if (rep == 2)
                printf("{\"probe\": \"%s\", \"h2d_GB\": %.3f, \"d2h_GB\": %.3f, \"ms\": %.2f, \"h2d_GBps\": %.1f, \"d2h_GBps\": %.1f}\n",
                       name, h2d / 1e9, d2h / 1e9, t * 1e3, h2d / t / 1e9, d2h / t / 1e9);
        }
        return 0;
    };
    run("h2d", n * 4, 0);
    run("d2h8", 0, n * 8);
    run("d2h4", 0, n * 4);
    run("d2h2", 0, n * 2);
    run("h2d4+d2h8", n * 4, n * 8);
    run("h2d4+d2h4", n * 4, n * 4);
    run("h2d4+d2h2", n * 4, n * 2);

    static int64_t table[65536];
    for (int i = 0; i < 65536; ++i) table[i] = (int64_t)i * 3 + 7;
    int Ts[] = {1, 2, 4, 8, 16, 32, 64};
    for (int T : Ts) {
        if (T > hw) break;
        // u16 code -> int64 via table, NT stores
        double best = 1e9, best32 = 1e9, bestc = 1e9;
        for (int rep = 0; rep < 3; ++rep) {
            double t = par(T, [&](int id, int TT) {
                size_t per = (n / TT + 7) & ~size_t(7), a = id * per, b = a + per < n ? a + per : n;
                for (size_t i = a; i + 8 <= b; i += 8) {
                    __m128i c = _mm_loadu_si128((const __m128i*)(hc16 + i));
                    __m512i idx = _mm512_cvtepu16_epi64(c);
                    __m512i v = _mm512_i64gather_epi64(idx, (const long long*)table, 8);
                    _mm512_stream_si512((__m512i*)(ho + i), v);
                }
            });
            best = t < best ? t : best;
            double t2 = par(T, [&](int id, int TT) {
                size_t per = (n / TT + 7) & ~size_t(7), a = id * per, b = a + per < n ? a + per : n;
                for (size_t i = a; i + 8 <= b; i += 8) {
                    __m256i c = _mm256_loadu_si256((const __m256i*)(hc32 + i));
                    _mm512_stream_si512((__m512i*)(ho + i), _mm512_cvtepu32_epi64(c));
                }
            });
            best32 = t2 < best32 ? t2 : best32;
            double t3 = par(T, [&](int id, int TT) {
                size_t per = (n / TT + 7) & ~size_t(7), a = id * per, b = a + per < n ? a + per : n;
                for (size_t i = a; i + 8 <= b; i += 8) _mm512_stream_si512((__m512i*)(ho + i), _mm512_set1_epi64(i));
            });
            bestc = t3 < bestc ? t3 : bestc;
        }
        printf("{\"probe\": \"host_widen\", \"threads\": %d, \"u16_table_ms\": %.2f, \"u32_widen_ms\": %.2f, \"nt_fill_ms\": %.2f, "
               "\"out_GBps_u16\": %.1f, \"out_GBps_u32\": %.1f, \"out_GBps_fill\": %.1f}\n",
               T, best * 1e3, best32 * 1e3, bestc * 1e3, n * 8 / best / 1e9, n * 8 / best32 / 1e9, n * 8 / bestc / 1e9);
        fflush(stdout);
    }
    // the combined pattern: D2H of 2-B codes + H2D of keys while host threads decode
    for (int T : {8, 16, 32}) {
        if (T > hw) break;
        CK(cudaDeviceSynchronize());
        double t0 = now();
        copies(dk, hk, n * 4, chunk, cudaMemcpyHostToDevice, s, 2);
        copies(hc16, do_, n * 2, chunk, cudaMemcpyDeviceToHost, s + 2, 2);
        double tc = par(T, [&](int id, int TT) {
            size_t per = (n / TT + 7) & ~size_t(7), a = id * per, b = a + per < n ? a + per : n;
            for (size_t i = a; i + 8 <= b; i += 8) {
                __m128i c = _mm_loadu_si128((const __m128i*)(hc16 + i));
                __m512i v = _mm512_i64gather_epi64(_mm512_cvtepu16_epi64(c), (const long long*)table, 8);
                _mm512_stream_si512((__m512i*)(ho + i), v);
            }
        });
        CK(cudaDeviceSynchronize());
        double t = now() - t0;
        printf("{\"probe\": \"concurrent_h2d4_d2h2_decode\", \"threads\": %d, \"ms\": %.2f, \"decode_ms\": %.2f}\n", T, t * 1e3, tc * 1e3);
    }
    return 0;
}
