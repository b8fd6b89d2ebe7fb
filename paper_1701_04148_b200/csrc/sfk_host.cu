// Point queries for a key batch in HOST memory (sfk_min_query_host): the
// reference's query_many (_kernels.py:229-241, sf.py:189-193) takes a host
// array and returns a host int64 array, so the PCIe link, not the GPU, bounds
// it. On a B200 box the x16 link moves ~55 GB/s per direction but only ~78 GB/s
// in both at once (profiles/r02/host_io_probe.jsonl), so int64 estimates
// (8 B per query back against 4 B of u32 keys in) make the return direction
// the bottleneck. Here the estimates cross the link narrowed and host threads
// widen them into the caller's int64 array:
//   * code16 (the default when the slim allows it): values below WIRE_BASE
//     travel as themselves, larger ones as WIRE_BASE + their index in the
//     slim's sorted distinct large values (at most WIRE_DICT of them). An
//     estimate is one of the slim's counter values, so this is exact;
//   * u32: every estimate as uint32 (counters are uint32);
//   * int64: the estimates as they are (also every `direct`-th chunk when the
//     output is pinned, to use the return direction's spare bandwidth).
// Chunks flow through three streams (H2D keys -> fused query kernel + narrow
// -> D2H) over a ring of device and pinned host slots while a host thread pool
// widens finished chunks with AVX-512 (scalar loop on CPUs without it).
#include <cuda_runtime.h>
#include <immintrin.h>

#include <algorithm>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/sfsketch_cuda.h"
#include "sfk_common.cuh"

namespace sfk {

int launch_min_query(const uint32_t*, const uint64_t*, int, int64_t, KeySrc, int64_t, int64_t*, cudaStream_t);

constexpr uint32_t WIRE_BASE = 0xF800u;
constexpr int WIRE_DICT = (int)(65536u - WIRE_BASE);  // 2048 large values
constexpr int DICT_SET_LOG = 12, DICT_SET = 1 << DICT_SET_LOG;  // device set of distinct large values

enum { WIRE_AUTO = 0, WIRE_I64 = 1, WIRE_U32 = 2, WIRE_C16 = 3 };

// ---------------------------------------------------------------- device side
// distinct counter values >= WIRE_BASE into an open-addressing set of
// DICT_SET slots (0 = empty: no large value is 0); *full is set when a value
// finds no slot (more distinct values than the set holds)
__global__ void dict_collect_k(const uint32_t* __restrict__ c, int64_t n, uint32_t* __restrict__ set,
                               unsigned* __restrict__ full) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t v = c[i];
    if (v < WIRE_BASE) continue;
    uint32_t h = (v * 0x9E3779B1u) >> (32 - DICT_SET_LOG);
    int p = 0;
    for (; p < DICT_SET; ++p, h = (h + 1) & (DICT_SET - 1)) {
      const uint32_t cur = *(volatile uint32_t*)(set + h);
      if (cur == v) break;
      if (cur == 0) {
        const uint32_t old = atomicCAS(set + h, 0u, v);
        if (old == 0u || old == v) break;
      }
    }
    if (p == DICT_SET) atomicExch(full, 1u);
  }
}

__device__ __forceinline__ uint32_t wire_code(uint32_t v, const uint32_t* sd, int nd) {
  if (v < WIRE_BASE) return v;
  int lo = 0, hi = nd;  // first index with sd[i] >= v (v is present)
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (sd[mid] < v) lo = mid + 1;
    else hi = mid;
  }
  return WIRE_BASE + (uint32_t)lo;
}

// int64 estimates -> u16 wire codes, 8 per thread and step (64 B in, 16 B out)
__global__ void __launch_bounds__(256) narrow16_k(const int64_t* __restrict__ est, int64_t n,
                                                  const uint32_t* __restrict__ dict, int nd,
                                                  uint16_t* __restrict__ out) {
  __shared__ uint32_t sd[WIRE_DICT];
  for (int i = threadIdx.x; i < nd; i += blockDim.x) sd[i] = dict[i];
  __syncthreads();
  const int64_t n8 = n >> 3, stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n8; g += stride) {
    const longlong2* p = reinterpret_cast<const longlong2*>(est) + g * 4;
    uint32_t c[8];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const longlong2 q = __ldcs(p + k);
      c[2 * k] = wire_code((uint32_t)q.x, sd, nd);
      c[2 * k + 1] = wire_code((uint32_t)q.y, sd, nd);
    }
    __stcs(reinterpret_cast<uint4*>(out) + g,
           make_uint4(c[0] | c[1] << 16, c[2] | c[3] << 16, c[4] | c[5] << 16, c[6] | c[7] << 16));
  }
  for (int64_t t = n8 * 8 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += stride)
    out[t] = (uint16_t)wire_code((uint32_t)est[t], sd, nd);
}

__global__ void __launch_bounds__(256) narrow32_k(const int64_t* __restrict__ est, int64_t n,
                                                  uint32_t* __restrict__ out) {
  const int64_t n4 = n >> 2, stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n4; g += stride) {
    const longlong2* p = reinterpret_cast<const longlong2*>(est) + g * 2;
    const longlong2 a = __ldcs(p), b = __ldcs(p + 1);
    __stcs(reinterpret_cast<uint4*>(out) + g, make_uint4((uint32_t)a.x, (uint32_t)a.y, (uint32_t)b.x, (uint32_t)b.y));
  }
  for (int64_t t = n4 * 4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += stride)
    out[t] = (uint32_t)est[t];
}

// ---------------------------------------------------------------- host widening
static bool has_avx512() {
  static const int ok = __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512bw") ? 1 : 0;
  return ok != 0;
}

static void widen16_scalar(const uint16_t* c, int64_t n, const int64_t* hi, int64_t* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = c[i] < WIRE_BASE ? (int64_t)c[i] : hi[c[i] - WIRE_BASE];
}
static void widen32_scalar(const uint32_t* c, int64_t n, int64_t* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = (int64_t)c[i];
}

// streaming (non-temporal) 64-B stores: the output is written once and is
// far larger than the caches
__attribute__((target("avx512f,avx512bw"))) static void widen16_avx512(const uint16_t* c, int64_t n,
                                                                       const int64_t* hi, int64_t* out) {
  int64_t i = 0;
  while (i < n && (reinterpret_cast<uintptr_t>(out + i) & 63)) {
    out[i] = c[i] < WIRE_BASE ? (int64_t)c[i] : hi[c[i] - WIRE_BASE];
    ++i;
  }
  const __m512i base = _mm512_set1_epi64(WIRE_BASE);
  for (; i + 8 <= n; i += 8) {
    const __m512i v = _mm512_cvtepu16_epi64(_mm_loadu_si128(reinterpret_cast<const __m128i*>(c + i)));
    const __mmask8 big = _mm512_cmpge_epu64_mask(v, base);
    __m512i r = v;
    if (big) r = _mm512_mask_i64gather_epi64(v, big, _mm512_sub_epi64(v, base), hi, 8);
    _mm512_stream_si512(reinterpret_cast<__m512i*>(out + i), r);
  }
  for (; i < n; ++i) out[i] = c[i] < WIRE_BASE ? (int64_t)c[i] : hi[c[i] - WIRE_BASE];
  _mm_sfence();
}
__attribute__((target("avx512f,avx512bw"))) static void widen32_avx512(const uint32_t* c, int64_t n, int64_t* out) {
  int64_t i = 0;
  while (i < n && (reinterpret_cast<uintptr_t>(out + i) & 63)) out[i] = (int64_t)c[i], ++i;
  for (; i + 8 <= n; i += 8)
    _mm512_stream_si512(reinterpret_cast<__m512i*>(out + i),
                        _mm512_cvtepu32_epi64(_mm256_loadu_si256(reinterpret_cast<const __m256i*>(c + i))));
  for (; i < n; ++i) out[i] = (int64_t)c[i];
  _mm_sfence();
}

// ---------------------------------------------------------------- thread pool
// run(f, T) calls f(id, T) for id < T on pool threads and the caller (id 0)
// and returns when all have finished. One pool of hardware-concurrency
// threads lives for the process; workers sleep on a condition variable.
class Pool {
 public:
  explicit Pool(int n) : n_(n < 1 ? 1 : n) {
    for (int i = 1; i < n_; ++i) th_.emplace_back([this, i] { loop(i); });
    for (auto& t : th_) t.detach();  // never joined: lives for the process
  }
  int size() const { return n_; }
  void run(const std::function<void(int, int)>& f, int T) {
    T = std::max(1, std::min(T, n_));
    std::lock_guard<std::mutex> one(run_mu_);  // one job at a time (callers on several devices)
    {
      std::lock_guard<std::mutex> g(mu_);
      job_ = &f;
      active_ = T;
      pending_ = T - 1;
      ++gen_;
    }
    if (T > 1) cv_.notify_all();
    f(0, T);
    std::unique_lock<std::mutex> g(mu_);
    done_.wait(g, [this] { return pending_ == 0; });
    job_ = nullptr;
  }

 private:
  void loop(int id) {
    unsigned long long seen = 0;
    for (;;) {
      const std::function<void(int, int)>* f;
      int T;
      {
        std::unique_lock<std::mutex> g(mu_);
        cv_.wait(g, [&] { return gen_ != seen; });
        seen = gen_;
        f = job_;
        T = active_;
      }
      if (id >= T) continue;  // not part of this job
      (*f)(id, T);
      std::lock_guard<std::mutex> g(mu_);
      if (--pending_ == 0) done_.notify_one();
    }
  }
  int n_;
  std::vector<std::thread> th_;
  std::mutex mu_, run_mu_;
  std::condition_variable cv_, done_;
  const std::function<void(int, int)>* job_ = nullptr;
  int active_ = 1;
  int pending_ = 0;
  unsigned long long gen_ = 0;
};

// [a, b) of `n` items for thread id of T, in multiples of 8 items
static inline void split(int64_t n, int id, int T, int64_t* a, int64_t* b) {
  const int64_t per = ((n + T - 1) / T + 7) & ~int64_t(7);
  *a = std::min<int64_t>(n, per * id);
  *b = std::min<int64_t>(n, *a + per);
}

// ---------------------------------------------------------------- configuration
static int64_t g_chunk = 1 << 22;  // keys per chunk (8 MiB of u16 codes: read back while still in the LLC)
static int64_t g_wire = WIRE_AUTO;
static int64_t g_direct = 0;      // every g_direct-th chunk returns int64 directly (pinned output only)
static int64_t g_threads = 0;     // 0: 3/4 of the hardware threads / local ranks (all of them contend with the DMA for host memory)
static int64_t g_ring = 8;        // chunks in flight
static int64_t g_last_wire = 0;
// the knobs are read once per call and may be set from any thread
static inline int64_t knob(const int64_t& k) { return __atomic_load_n(&k, __ATOMIC_RELAXED); }

// ---------------------------------------------------------------- per-device state
struct Slot {
  void* dkeys = nullptr;
  int64_t* dest = nullptr;
  void* dwire = nullptr;
  void* hwire = nullptr;  // pinned
  void* hkeys = nullptr;  // pinned key staging for pageable input
  cudaEvent_t e_h2d = nullptr, e_comp = nullptr, e_d2h = nullptr;
};

struct HostQ {
  int dev = -1;
  cudaStream_t sh = nullptr, sc = nullptr, sd = nullptr;
  int64_t chunk = 0, kbytes = 0;
  std::vector<Slot> slots;
  uint32_t *dlist = nullptr, *ddict = nullptr;  // the device set of large values; the sorted dictionary
  unsigned* dcnt = nullptr;                     // set-full flag
  uint32_t* hlist = nullptr;                    // pinned: [full flag][set...], then the dictionary upload
  cudaEvent_t e_start = nullptr;
  std::mutex mu;

  void release_slots() {
    for (auto& s : slots) {
      cudaFree(s.dkeys);
      cudaFree(s.dest);
      cudaFree(s.dwire);
      cudaFreeHost(s.hwire);
      cudaFreeHost(s.hkeys);
      cudaEventDestroy(s.e_h2d);
      cudaEventDestroy(s.e_comp);
      cudaEventDestroy(s.e_d2h);
    }
    slots.clear();
    chunk = kbytes = 0;
  }
  int init(int device) {
    dev = device;
    if (cudaStreamCreateWithFlags(&sh, cudaStreamNonBlocking) || cudaStreamCreateWithFlags(&sc, cudaStreamNonBlocking) ||
        cudaStreamCreateWithFlags(&sd, cudaStreamNonBlocking) || cudaEventCreateWithFlags(&e_start, cudaEventDisableTiming) ||
        cudaMalloc(&dlist, DICT_SET * 4) || cudaMalloc(&ddict, WIRE_DICT * 4) || cudaMalloc(&dcnt, 4) ||
        cudaHostAlloc(&hlist, (DICT_SET + 1) * 4, 0)) {
      set_error("sfk_min_query_host setup: %s", cudaGetErrorString(cudaGetLastError()));
      return 1;
    }
    return 0;
  }
  // ring of `ring` slots holding at least `ch` keys of `esz` bytes each
  int ensure(int64_t ch, int64_t esz, int ring) {
    if ((int)slots.size() == ring && chunk >= ch && kbytes >= ch * esz) return 0;
    // the old slots may still be in use on this context's streams
    cudaStreamSynchronize(sh);
    cudaStreamSynchronize(sc);
    cudaStreamSynchronize(sd);
    release_slots();
    slots.resize(ring);
    for (auto& s : slots) {
      if (cudaMalloc(&s.dkeys, ch * esz) || cudaMalloc(&s.dest, ch * 8) || cudaMalloc(&s.dwire, ch * 4) ||
          cudaHostAlloc(&s.hwire, ch * 4, 0) || cudaHostAlloc(&s.hkeys, ch * esz, 0) ||
          cudaEventCreateWithFlags(&s.e_h2d, cudaEventDisableTiming) ||
          cudaEventCreateWithFlags(&s.e_comp, cudaEventDisableTiming) ||
          cudaEventCreateWithFlags(&s.e_d2h, cudaEventDisableTiming)) {
        set_error("sfk_min_query_host buffers (%lld keys x %d): %s", (long long)ch, ring,
                  cudaGetErrorString(cudaGetLastError()));
        release_slots();
        return 1;
      }
    }
    chunk = ch;
    kbytes = ch * esz;
    return 0;
  }
};

static std::mutex g_ctx_mu;
static std::vector<HostQ*> g_ctx;
static Pool* g_pool = nullptr;

static HostQ* ctx_for(int dev) {
  std::lock_guard<std::mutex> g(g_ctx_mu);
  if ((int)g_ctx.size() <= dev) g_ctx.resize(dev + 1, nullptr);
  if (!g_ctx[dev]) {
    HostQ* q = new HostQ();
    if (q->init(dev)) {
      delete q;
      return nullptr;
    }
    g_ctx[dev] = q;
  }
  if (!g_pool) g_pool = new Pool(std::max(1, (int)std::thread::hardware_concurrency()));
  return g_ctx[dev];
}

static bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// sorted distinct counter values >= WIRE_BASE of the slim; *ok = false if
// there are more than WIRE_DICT (the code16 wire does not apply)
static int build_dict(HostQ* q, const uint32_t* counters, int64_t cells, std::vector<uint32_t>* dict, bool* ok) {
  cudaMemsetAsync(q->dlist, 0, DICT_SET * 4, q->sc);
  cudaMemsetAsync(q->dcnt, 0, 4, q->sc);
  note_launch();
  dict_collect_k<<<grid_for(cells, 256, sm_count() * 4), 256, 0, q->sc>>>(counters, cells, q->dlist, q->dcnt);
  if (int rc = check_launch("dict_collect_k")) return rc;
  cudaMemcpyAsync(q->hlist, q->dcnt, 4, cudaMemcpyDeviceToHost, q->sc);
  cudaMemcpyAsync(q->hlist + 1, q->dlist, DICT_SET * 4, cudaMemcpyDeviceToHost, q->sc);
  if (cudaStreamSynchronize(q->sc) != cudaSuccess) {
    set_error("sfk_min_query_host dict: %s", cudaGetErrorString(cudaGetLastError()));
    return 1;
  }
  *ok = false;
  dict->clear();
  if (q->hlist[0]) return 0;
  for (int k = 1; k <= DICT_SET; ++k)
    if (q->hlist[k]) dict->push_back(q->hlist[k]);
  std::sort(dict->begin(), dict->end());
  if ((int)dict->size() > WIRE_DICT) return 0;
  *ok = true;
  return 0;
}

}  // namespace sfk

using namespace sfk;

extern "C" {

int64_t sfk_host_query_config(int what, int64_t value) {
  int64_t* k = what == 0 ? &g_chunk : what == 1 ? &g_wire : what == 2 ? &g_direct : what == 3 ? &g_threads
             : what == 4 ? &g_ring : what == 5 ? &g_last_wire : nullptr;
  if (!k) return -1;
  if (value < 0 || what == 5) return knob(*k);
  if (what == 0) value = std::max<int64_t>(4096, (value + 4095) & ~int64_t(4095));
  if (what == 4) value = std::min<int64_t>(16, std::max<int64_t>(2, value));
  if (what == 1 && value > WIRE_C16) return -1;
  return __atomic_exchange_n(k, value, __ATOMIC_RELAXED);
}

int sfk_min_query_host_staged(const uint32_t*, const uint64_t*, int, int64_t, const void*, int, int, int64_t, int64_t*,
                              const void*, int64_t, void*);

int sfk_min_query_host(const uint32_t* counters, const uint64_t* seeds, int d, int64_t w, const void* keys_host,
                       int key_kind, int rec_len, int64_t n, int64_t* out_host, void* stream) {
  return sfk_min_query_host_staged(counters, seeds, d, w, keys_host, key_kind, rec_len, n, out_host, nullptr, 0,
                                   stream);
}

// keys_dev: the batch's first n_dev keys already resident on the device (a
// copy of keys_host's prefix, ordered before `stream`'s work): chunks that lie
// wholly inside it are queried in place, with no H2D.
int sfk_min_query_host_staged(const uint32_t* counters, const uint64_t* seeds, int d, int64_t w,
                              const void* keys_host, int key_kind, int rec_len, int64_t n, int64_t* out_host,
                              const void* keys_dev, int64_t n_dev, void* stream) {
  if (d < 1 || d > MAXSEEDS || w < 1 || (uint64_t)d * (uint64_t)w >= (1ull << 32)) {
    set_error("sfk_min_query_host: bad sketch shape d=%d w=%lld", d, (long long)w);
    return 1;
  }
  if (key_kind != SFK_KEY_U32 && key_kind != SFK_KEY_U64 && !(key_kind == SFK_KEY_RECORD && rec_len >= 1)) {
    set_error("sfk_min_query_host: unknown key kind %d", key_kind);
    return 1;
  }
  if (n < 0 || (n > 0 && (!keys_host || !out_host))) {
    set_error("sfk_min_query_host: bad arguments");
    return 1;
  }
  if (n_dev < 0 || (n_dev > 0 && !keys_dev)) {
    set_error("sfk_min_query_host: bad staged keys");
    return 1;
  }
  if (n == 0) return 0;
  n_dev = std::min(n_dev, n);
  int dev = 0;
  cudaGetDevice(&dev);
  HostQ* q = ctx_for(dev);
  if (!q) return 1;
  std::lock_guard<std::mutex> guard(q->mu);
  const int64_t esz = key_kind == SFK_KEY_U32 ? 4 : key_kind == SFK_KEY_U64 ? 8 : rec_len;
  const int ring = (int)knob(g_ring);
  const int64_t C = std::min<int64_t>(knob(g_chunk), (n + 4095) & ~int64_t(4095));
  if (q->ensure(C, esz, ring)) return 1;
  const int64_t CH = C;
  const bool keys_pinned = is_pinned(keys_host), out_pinned = is_pinned(out_host);
  cudaStream_t caller = (cudaStream_t)stream;
  cudaEventRecord(q->e_start, caller);
  cudaStreamWaitEvent(q->sh, q->e_start, 0);
  cudaStreamWaitEvent(q->sc, q->e_start, 0);

  // wire format
  int wire = (int)knob(g_wire);
  const int64_t direct_every = knob(g_direct);
  std::vector<uint32_t> dict;
  std::vector<int64_t> hi;
  if (wire == WIRE_AUTO || wire == WIRE_C16) {
    bool ok = false;
    if (int rc = build_dict(q, counters, (int64_t)d * w, &dict, &ok)) return rc;
    if (ok) {
      wire = WIRE_C16;
      if (!dict.empty()) {
        memcpy(q->hlist, dict.data(), dict.size() * 4);
        cudaMemcpyAsync(q->ddict, q->hlist, dict.size() * 4, cudaMemcpyHostToDevice, q->sc);
      }
      hi.assign(WIRE_DICT, 0);
      for (size_t k = 0; k < dict.size(); ++k) hi[k] = (int64_t)dict[k];
    } else {
      wire = WIRE_U32;
    }
  }
  __atomic_store_n(&g_last_wire, (int64_t)wire, __ATOMIC_RELAXED);
  const int nd = (int)dict.size();
  const int64_t wb = wire == WIRE_C16 ? 2 : wire == WIRE_U32 ? 4 : 8;
  const int64_t nc = (n + CH - 1) / CH;
  auto direct = [&](int64_t j) {
    return wire == WIRE_I64 || (out_pinned && direct_every > 0 && j % direct_every == direct_every - 1);
  };
  Pool& pool = *g_pool;
  // threads: the knob, else 3/4 of the hardware threads shared among the
  // node's ranks (torchrun's LOCAL_WORLD_SIZE), so N processes do not
  // oversubscribe the host
  int ranks = 1;
  if (const char* lw = getenv("LOCAL_WORLD_SIZE")) ranks = std::max(1, atoi(lw));
  const int64_t gt = knob(g_threads);
  const int T = std::max(1, gt > 0 ? (int)gt : pool.size() * 3 / 4 / ranks);
  const bool avx = has_avx512();
  int rc = 0;

  auto enqueue = [&](int64_t j) -> int {
    Slot& s = q->slots[j % ring];
    const int64_t a = j * CH, m = std::min(CH, n - a);
    const char* src = static_cast<const char*>(keys_host) + a * esz;
    const bool staged = a + m <= n_dev;
    const void* kdev = staged ? static_cast<const char*>(keys_dev) + a * esz : s.dkeys;
    if (staged) {
      // already resident: no copy; the query still waits for the slot's last D2H
    } else {
    if (j >= ring) cudaStreamWaitEvent(q->sh, s.e_comp, 0);  // key slot free
    if (!keys_pinned) {
      if (j >= ring) cudaEventSynchronize(s.e_h2d);  // pinned staging slot free
      char* dst = static_cast<char*>(s.hkeys);
      const int64_t bytes = m * esz;
      pool.run([&](int id, int TT) {
        int64_t x, y;
        split(bytes, id, TT, &x, &y);
        if (y > x) memcpy(dst + x, src + x, y - x);
      }, T);
      src = dst;
    }
    cudaMemcpyAsync(s.dkeys, src, m * esz, cudaMemcpyHostToDevice, q->sh);
    cudaEventRecord(s.e_h2d, q->sh);
    cudaStreamWaitEvent(q->sc, s.e_h2d, 0);
    }
    if (j >= ring) cudaStreamWaitEvent(q->sc, s.e_d2h, 0);  // dest / wire slot free
    if (int r = launch_min_query(counters, seeds, d, w, KeySrc{kdev, key_kind, rec_len}, m, s.dest, q->sc))
      return r;
    if (!direct(j)) {
      note_launch();
      const int grid = grid_for(m, 256 * 8, sm_count() * 4);
      if (wire == WIRE_C16)
        narrow16_k<<<grid, 256, 0, q->sc>>>(s.dest, m, q->ddict, nd, static_cast<uint16_t*>(s.dwire));
      else
        narrow32_k<<<grid, 256, 0, q->sc>>>(s.dest, m, static_cast<uint32_t*>(s.dwire));
      if (int r = check_launch("narrow_k")) return r;
    }
    cudaEventRecord(s.e_comp, q->sc);
    cudaStreamWaitEvent(q->sd, s.e_comp, 0);
    if (direct(j))
      cudaMemcpyAsync(out_host + a, s.dest, m * 8, cudaMemcpyDeviceToHost, q->sd);
    else
      cudaMemcpyAsync(s.hwire, s.dwire, m * wb, cudaMemcpyDeviceToHost, q->sd);
    cudaEventRecord(s.e_d2h, q->sd);
    return 0;
  };

  int64_t next = 0;
  for (; next < std::min<int64_t>(ring, nc) && !rc; ++next) rc = enqueue(next);
  for (int64_t c = 0; c < nc && !rc; ++c) {
    Slot& s = q->slots[c % ring];
    if (cudaEventSynchronize(s.e_d2h) != cudaSuccess) {
      set_error("sfk_min_query_host: %s", cudaGetErrorString(cudaGetLastError()));
      rc = 1;
      break;
    }
    if (!direct(c)) {
      const int64_t a = c * CH, m = std::min(CH, n - a);
      int64_t* o = out_host + a;
      const void* hw = s.hwire;
      const int64_t* hp = hi.data();
      pool.run([&](int id, int TT) {
        int64_t x, y;
        split(m, id, TT, &x, &y);
        if (y <= x) return;
        if (wire == WIRE_C16) {
          const uint16_t* cc = static_cast<const uint16_t*>(hw) + x;
          if (avx) widen16_avx512(cc, y - x, hp, o + x);
          else widen16_scalar(cc, y - x, hp, o + x);
        } else {
          const uint32_t* cc = static_cast<const uint32_t*>(hw) + x;
          if (avx) widen32_avx512(cc, y - x, o + x);
          else widen32_scalar(cc, y - x, o + x);
        }
      }, T);
    }
    if (next < nc) rc = enqueue(next++);
  }
  if (rc) {
    cudaStreamSynchronize(q->sh);
    cudaStreamSynchronize(q->sc);
    cudaStreamSynchronize(q->sd);
  }
  return rc;
}

}  // extern "C"
