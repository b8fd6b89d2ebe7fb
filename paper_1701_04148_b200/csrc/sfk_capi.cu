// extern "C" entry points of libsfsketch_cuda.so (declared in
// include/sfsketch_cuda.h). Each one validates its arguments, picks the
// parallel engine or the exact sequential device engine, and splits very
// large batches into chunks the 32-bit pair encoding can address.
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <cmath>

#include "sfk_common.cuh"

namespace sfk {

static thread_local char g_err[512] = "";
static unsigned long long g_launches = 0;

void note_launch() { __atomic_fetch_add(&g_launches, 1ull, __ATOMIC_RELAXED); }

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int check_launch(const char* where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", where, cudaGetErrorString(e));
    return (int)e;
  }
  return 0;
}

int sm_count() {
  static int sms[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!sms[dev]) {
    cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev);
    if (sms[dev] < 1) sms[dev] = 1;
  }
  return sms[dev];
}

// implemented in sfk_query.cu / sfk_seq.cu / sfk_sf.cu
int launch_min_query(const uint32_t*, const uint64_t*, int, int64_t, KeySrc, int64_t, int64_t*, cudaStream_t);
int launch_mix_batch(const uint64_t*, int64_t, uint64_t*, cudaStream_t);
int query_path(int mode);
int launch_query_index(const uint64_t*, int, int64_t, KeySrc, int64_t, uint16_t*, cudaStream_t);
int launch_min_query_idx(const uint32_t*, int, int64_t, const uint16_t*, int64_t, int64_t*, cudaStream_t);
int query_last_path();
int launch_load_keys(KeySrc, int64_t, uint64_t*, cudaStream_t);
int launch_gen_query_keys(uint64_t, const uint32_t*, const uint32_t*, uint32_t, const double*, int64_t, int64_t,
                          uint32_t*, cudaStream_t);
int launch_seq_apply(int kind, int variant, uint32_t* slim, uint32_t* fat, uint32_t* dsub, const uint64_t* s_seeds,
                     const uint64_t* f_seeds, int d, int64_t w, int64_t wp, int64_t z, const uint8_t* ops, KeySrc ks,
                     const int64_t* true_counts, int64_t n, int64_t* inc, int64_t* result, cudaStream_t st);
int launch_blk_bucket(int variant, uint32_t* slim, uint32_t* fat, const uint64_t* s_seeds, const uint64_t* f_seeds,
                      int d, int64_t w, int64_t z, const uint8_t* ops, KeySrc ks, int64_t n, int64_t* inc,
                      int64_t* result, cudaStream_t st);
bool blk_fits(int d, int64_t w, int64_t z, int64_t n);
int blk_profile(unsigned long long* out);
int launch_seqw_bucket(int variant, uint32_t* slim, uint32_t* fat, const uint64_t* s_seeds, const uint64_t* f_seeds,
                       int d, int64_t w, int64_t z, const uint8_t* ops, KeySrc ks, int64_t n, int64_t* inc,
                       int64_t* result, cudaStream_t st);
size_t parallel_workspace_size(int kind, int d, int64_t w, int64_t wp, int z, int64_t n);
int engine_stats(unsigned long long* out, int reset);
int engine_timing(int on);
int engine_trace(unsigned long long* host_out, size_t runs);
float engine_last_ms();
int parallel_apply(int kind, uint32_t* slim, uint32_t* fat, uint32_t* dsub, const uint64_t* slim_seeds,
                   const uint64_t* fat_seeds, int d, int64_t w, int64_t wp, int z, const uint8_t* ops, KeySrc ks,
                   int64_t n, int64_t* inc, int64_t* result, void* ws, size_t ws_bytes, cudaStream_t st,
                   const ExtArgs* ext = nullptr);
int collect_stats(const uint8_t* ops, int64_t n, const uint32_t* counters, int64_t cells, void* ws, size_t ws_bytes,
                  Stats* host, cudaStream_t st, uint32_t bias = 0);
int count_fast(int32_t* counters, const uint64_t* seeds, int d, int64_t w, const uint8_t* ops, KeySrc ks, int64_t n,
               cudaStream_t st);
int ext_query(int which, const void* table, const uint64_t* seeds, int d, int64_t w, KeySrc ks, int64_t n,
              const int64_t* vtab, int64_t* out, cudaStream_t st);
int launch_pcg_uniform(uint64_t sh, uint64_t sl, uint64_t ih, uint64_t il, int64_t offset, int64_t n,
                       const double* cdf, int64_t v, int64_t* ranks, double* uout, cudaStream_t st);
size_t pcg_bounded_workspace_size(int64_t n, int64_t v);
int launch_pcg_bounded(uint64_t sh, uint64_t sl, uint64_t ih, uint64_t il, int64_t offset64, int64_t n, int64_t v,
                       int64_t* out, int64_t* next_offset64, void* ws, size_t ws_bytes, cudaStream_t st);
int launch_interleave(const int64_t* cand, const double* decide, const double* pick, double p, int64_t n, int64_t v,
                      uint8_t* ops, int64_t* ranks, void* ws, size_t ws_bytes, cudaStream_t st);
size_t trace_workspace_size(int64_t nb);
int trace_parse_lines(const uint8_t* txt, int64_t nb, int64_t* line_pos, uint8_t* status, uint8_t* lop, uint64_t* lkey,
                      int64_t* out_info, void* ws, size_t ws_bytes, cudaStream_t st);
int trace_compact(const uint8_t* status, const uint8_t* lop, const uint64_t* lkey, int64_t nlines, uint8_t* ops,
                  uint64_t* keys, int64_t* out_n, void* ws, size_t ws_bytes, int64_t nb, cudaStream_t st);
int gated_precheck(const int64_t* tc, int64_t n, const double* gate, const uint16_t* exps, const uint32_t* slim,
                   int64_t cells, void* ws, size_t ws_bytes, bool* ok, cudaStream_t st);
int launch_seq_ext(int kind, void* counters, const uint64_t* seeds, int d, int64_t w, const uint8_t* ops, KeySrc ks,
                   int64_t n, const double* gate, uint64_t rng_seed, int64_t start_pos, int64_t* result,
                   cudaStream_t st);
int cm_fast(uint32_t* counters, const uint64_t* seeds, int d, int64_t w, const uint8_t* ops, KeySrc ks, int64_t n,
            cudaStream_t st);

__global__ void set_result_k(int64_t* result, int64_t status, int64_t idx, int64_t n_ins, int64_t* inc, int d,
                             int64_t inc_add) {
  result[0] = status;
  result[1] = idx;
  result[2] = n_ins;
  if (inc)
    for (int i = 0; i < d; ++i) inc[i] += inc_add;
}

// parallel kinds (sfk_sf.cu): 0 SFF, 1 SF1, 2 CU, 3 CM exact
#ifndef SFK_SMALL_BATCH_DEFAULT
#define SFK_SMALL_BATCH_DEFAULT 32
#endif

static int64_t chunk_ops(int d, int z) {
  // t << (kb + 1) must fit 32 bits and d * n must fit a signed int
  int kb = 0;
  while ((1 << kb) < std::max(z, 1)) ++kb;
  int64_t lim_t = (int64_t)1 << (31 - kb);
  int64_t lim_n = ((int64_t)1 << 30) / std::max(d, 1);
  return std::min(lim_t, lim_n);
}

// Batches of at most this many ops run on the exact one-thread device engine:
// one launch and no host round trip, against ~17-24 launches (plus CUB's)
// and, for CM / CU, a precheck read-back on the parallel pipeline, whose
// fixed cost (~80-140 us per batch) dominates tiny batches such as the
// reference's insert(key) / delete(key). sfk_small_batch_ops() sets it (0: off).
static int64_t g_small_batch = SFK_SMALL_BATCH_DEFAULT;
static int64_t small_batch_ops() { return __atomic_load_n(&g_small_batch, __ATOMIC_RELAXED); }

static bool small_batch(int64_t n) { return n > 0 && n <= small_batch_ops(); }

// SFF / SF4 batches up to this many ops run on the warp-cooperative exact
// engine (seqw_bucket_k): one launch, no host round trip, ~0.1-0.3 us per op
// instead of the parallel pipeline's ~140 us fixed cost. sfk_warp_batch_ops()
// sets it (0: off).
#ifndef SFK_WARP_BATCH_DEFAULT
#define SFK_WARP_BATCH_DEFAULT 24
#endif
static int64_t g_warp_batch = SFK_WARP_BATCH_DEFAULT;
static int64_t warp_batch_ops() { return __atomic_load_n(&g_warp_batch, __ATOMIC_RELAXED); }

// Larger SFF / SF4 batches up to this many ops (and d x n <= 8192 (op, row)
// pairs) run on the block engine (blk_bucket_k, sfk_blk.cu): one 1024-thread
// CTA, sort + fat walk + dataflow replay in shared memory, one launch.
// sfk_block_batch_ops() sets it (0: off).
#ifndef SFK_BLOCK_BATCH_DEFAULT
#define SFK_BLOCK_BATCH_DEFAULT 2048
#endif
static int64_t g_block_batch = SFK_BLOCK_BATCH_DEFAULT;
static int64_t block_batch_ops() { return __atomic_load_n(&g_block_batch, __ATOMIC_RELAXED); }

static const char* key_ptr(const void* keys, int key_kind, int rec_len, int64_t t0) {
  const char* p = static_cast<const char*>(keys);
  int64_t sz = key_kind == SFK_KEY_U64 ? 8 : key_kind == SFK_KEY_U32 ? 4 : rec_len;
  return p + t0 * sz;
}

static int check_common(int d, int64_t w, int key_kind, int rec_len) {
  if (d < 1 || d > MAXSEEDS) { set_error("d must lie in [1, %d], got %d", MAXSEEDS, d); return 1; }
  if (w < 1 || (uint64_t)d * (uint64_t)w >= (1ull << 32)) { set_error("bad width w=%lld", (long long)w); return 1; }
  if (key_kind != SFK_KEY_U64 && key_kind != SFK_KEY_U32 && key_kind != SFK_KEY_RECORD) {
    set_error("unknown key kind %d", key_kind);
    return 1;
  }
  if (key_kind == SFK_KEY_RECORD && rec_len < 1) { set_error("record keys need rec_len >= 1"); return 1; }
  return 0;
}

// A batch split into several chunks is checked for bad op codes (anything
// but 0 / 1) before the first chunk runs, so a rejected batch applies
// nothing; single-chunk batches are checked on the device inside the apply.
static int bad_ops_first(const uint8_t* ops, int64_t n, int64_t chunk, void* ws, size_t ws_bytes, int64_t* result,
                         cudaStream_t st, bool* rejected) {
  *rejected = false;
  if (n <= chunk) return 0;
  Stats s;
  if (int r = collect_stats(ops, n, nullptr, 0, ws, ws_bytes, &s, st)) return r;
  if (s.first_bad < (unsigned long long)n) {
    *rejected = true;
    { note_launch(); set_result_k<<<1, 1, 0, st>>>(result, SFK_BAD_OPCODE, (int64_t)s.first_bad, 0, nullptr, 0, 0); }
    return check_launch("set_result");
  }
  return 0;
}

// Run `body(t0, cnt, result)` over chunks; accumulate {status, op_index, n_ins}.
template <typename F>
static int chunked(int64_t n, int64_t chunk, int64_t* result, cudaStream_t st, F body) {
  if (n <= 0) {
    { note_launch(); set_result_k<<<1, 1, 0, st>>>(result, SFK_OK, -1, 0, nullptr, 0, 0); }
    return check_launch("set_result");
  }
  if (n <= chunk) return body((int64_t)0, n);
  int64_t total_ins = 0;
  for (int64_t t0 = 0; t0 < n; t0 += chunk) {
    const int64_t cnt = std::min(chunk, n - t0);
    if (int r = body(t0, cnt)) return r;
    int64_t h[3];
    cudaMemcpyAsync(h, result, sizeof(h), cudaMemcpyDeviceToHost, st);
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) { set_error("chunk sync: %s", cudaGetErrorString(e)); return (int)e; }
    total_ins += h[2];
    if (h[0] != SFK_OK) {
      { note_launch(); set_result_k<<<1, 1, 0, st>>>(result, h[0], t0 + h[1], total_ins, nullptr, 0, 0); }
      return check_launch("set_result");
    }
  }
  { note_launch(); set_result_k<<<1, 1, 0, st>>>(result, SFK_OK, -1, total_ins, nullptr, 0, 0); }
  return check_launch("set_result");
}

}  // namespace sfk

using namespace sfk;

extern "C" {

int sfk_abi_version(void) { return 1; }

unsigned long long sfk_launch_count(void) { return __atomic_load_n(&g_launches, __ATOMIC_RELAXED); }

int sfk_engine_stats(unsigned long long* out8, int reset) { return engine_stats(out8, reset); }

int sfk_engine_timing(int on) { return engine_timing(on); }

int sfk_query_path(int mode) { return query_path(mode); }

int sfk_query_index(const uint64_t* seeds, int d, int64_t w, const void* keys, int key_kind, int rec_len, int64_t n,
                    uint16_t* idx, void* stream) {
  if (check_common(d, w, key_kind, rec_len)) return 1;
  return launch_query_index(seeds, d, w, KeySrc{keys, key_kind, rec_len}, n, idx, (cudaStream_t)stream);
}

int sfk_min_query_idx(const uint32_t* counters, int d, int64_t w, const uint16_t* idx, int64_t n, int64_t* out,
                      void* stream) {
  if (d < 1 || d > MAXSEEDS || w < 1) {
    set_error("bad sketch shape d=%d w=%lld", d, (long long)w);
    return 1;
  }
  return launch_min_query_idx(counters, d, w, idx, n, out, (cudaStream_t)stream);
}

int sfk_query_last_path(void) { return query_last_path(); }

int sfk_engine_trace(unsigned long long* host_out, size_t runs) { return engine_trace(host_out, runs); }

float sfk_engine_last_ms(void) { return engine_last_ms(); }

int sfk_gen_query_keys(uint64_t seed, const uint32_t* present, const uint32_t* sorted_present, uint32_t v,
                       const double* cdf, int64_t t0, int64_t n, uint32_t* out, void* stream) {
  return launch_gen_query_keys(seed, present, sorted_present, v, cdf, t0, n, out, (cudaStream_t)stream);
}

const char* sfk_last_error(void) { return g_err; }

int sfk_stream_sync(void* stream) {
  const cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) {
    set_error("stream sync: %s", cudaGetErrorString(e));
    return (int)e;
  }
  return 0;
}

int64_t sfk_small_batch_ops(int64_t ops) {
  return ops < 0 ? small_batch_ops() : __atomic_exchange_n(&g_small_batch, ops, __ATOMIC_RELAXED);
}

int64_t sfk_warp_batch_ops(int64_t ops) {
  return ops < 0 ? warp_batch_ops() : __atomic_exchange_n(&g_warp_batch, ops, __ATOMIC_RELAXED);
}

int sfk_blk_profile(unsigned long long* out) { return blk_profile(out); }

int64_t sfk_block_batch_ops(int64_t ops) {
  return ops < 0 ? block_batch_ops() : __atomic_exchange_n(&g_block_batch, ops, __ATOMIC_RELAXED);
}

int sfk_mix_batch(const uint64_t* keys, int64_t n, uint64_t* out, void* stream) {
  return launch_mix_batch(keys, n, out, (cudaStream_t)stream);
}

int sfk_load_keys(const void* keys, int key_kind, int rec_len, int64_t n, uint64_t* out, void* stream) {
  if (check_common(1, 1, key_kind, rec_len)) return 1;
  return launch_load_keys(KeySrc{keys, key_kind, rec_len}, n, out, (cudaStream_t)stream);
}

int sfk_min_query(const uint32_t* counters, const uint64_t* seeds, int d, int64_t w, const void* keys, int key_kind,
                  int rec_len, int64_t n, int64_t* out, void* stream) {
  if (check_common(d, w, key_kind, rec_len)) return 1;
  return launch_min_query(counters, seeds, d, w, KeySrc{keys, key_kind, rec_len}, n, out, (cudaStream_t)stream);
}

size_t sfk_cm_workspace_size(int d, int64_t w, int64_t n) {
  if (d > MAXD) return 256;
  return parallel_workspace_size(3, d, w, 0, 1, std::min<int64_t>(n, chunk_ops(d, 1)));
}

int sfk_cm_apply(uint32_t* counters, const uint64_t* seeds, int d, int64_t w, const uint8_t* ops, const void* keys,
                 int key_kind, int rec_len, int64_t n, int64_t* inc_counts, int64_t* result, void* workspace,
                 size_t workspace_bytes, int flags, void* stream) {
  if (check_common(d, w, key_kind, rec_len)) return 1;
  cudaStream_t st = (cudaStream_t)stream;
  if ((flags & SFK_FLAG_SEQUENTIAL) || d > MAXD || small_batch(n))
    return launch_seq_apply(0, 0, counters, nullptr, nullptr, seeds, nullptr, d, w, 0, 1, ops,
                            KeySrc{keys, key_kind, rec_len}, nullptr, n, inc_counts, result, st);
  bool rejected = false;
  if (int r = bad_ops_first(ops, n, chunk_ops(d, 1), workspace, workspace_bytes, result, st, &rejected)) return r;
  if (rejected) return 0;
  return chunked(n, chunk_ops(d, 1), result, st, [&](int64_t t0, int64_t cnt) -> int {
    KeySrc ks{key_ptr(keys, key_kind, rec_len, t0), key_kind, rec_len};
    Stats s;
    if (int r = collect_stats(ops + t0, cnt, counters, (int64_t)d * w, workspace, workspace_bytes, &s, st)) return r;
    if (s.first_bad < (unsigned long long)cnt) {  // reject the batch: nothing applied
      { note_launch(); set_result_k<<<1, 1, 0, st>>>(result, SFK_BAD_OPCODE, (int64_t)s.first_bad, 0, nullptr, 0, 0); }
      return check_launch("set_result");
    }
    // no insert can meet a saturated counter and no delete a zero one
    const bool safe = ((uint64_t)s.cmax + s.n_ins <= 0xFFFFFFFFull) && (s.n_del == 0 || (uint64_t)s.cmin >= s.n_del);
    if (safe) {
      if (int r = cm_fast(counters, seeds, d, w, ops + t0, ks, cnt, st)) return r;
      { note_launch(); set_result_k<<<1, 1, 0, st>>>(result, SFK_OK, -1, (int64_t)s.n_ins, inc_counts, d, (int64_t)s.n_ins); }
      return check_launch("set_result");
    }
    return parallel_apply(3, counters, nullptr, nullptr, seeds, nullptr, d, w, 0, 1, ops + t0, ks, cnt, inc_counts,
                          result, workspace, workspace_bytes, st);
  });
}

int sfk_cm_delta(uint32_t* counters, const uint64_t* seeds, int d, int64_t w, const uint8_t* ops, const void* keys,
                 int key_kind, int rec_len, int64_t n, void* stream) {
  if (check_common(d, w, key_kind, rec_len)) return 1;
  if (d > MAXD) {
    set_error("sfk_cm_delta: d=%d exceeds %d", d, MAXD);
    return 1;
  }
  if (n <= 0) return 0;
  return cm_fast(counters, seeds, d, w, ops, KeySrc{keys, key_kind, rec_len}, n, (cudaStream_t)stream);
}

size_t sfk_cu_workspace_size(int d, int64_t w, int64_t n) {
  if (d > MAXD) return 256;
  return parallel_workspace_size(2, d, w, 0, 1, std::min<int64_t>(n, chunk_ops(d, 1)));
}

int sfk_cu_apply(uint32_t* counters, const uint64_t* seeds, int d, int64_t w, const uint8_t* ops, const void* keys,
                 int key_kind, int rec_len, int64_t n, int64_t* inc_counts, int64_t* result, void* workspace,
                 size_t workspace_bytes, int flags, void* stream) {
  if (check_common(d, w, key_kind, rec_len)) return 1;
  cudaStream_t st = (cudaStream_t)stream;
  KeySrc all{keys, key_kind, rec_len};
  if ((flags & SFK_FLAG_SEQUENTIAL) || d > MAXD || small_batch(n))
    return launch_seq_apply(1, 0, counters, nullptr, nullptr, seeds, nullptr, d, w, 0, 1, ops, all, nullptr, n,
                            inc_counts, result, st);
  bool rejected = false;
  if (int r = bad_ops_first(ops, n, chunk_ops(d, 1), workspace, workspace_bytes, result, st, &rejected)) return r;
  if (rejected) return 0;
  return chunked(n, chunk_ops(d, 1), result, st, [&](int64_t t0, int64_t cnt) -> int {
    KeySrc ks{key_ptr(keys, key_kind, rec_len, t0), key_kind, rec_len};
    Stats s;
    if (int r = collect_stats(ops + t0, cnt, counters, (int64_t)d * w, workspace, workspace_bytes, &s, st)) return r;
    if (s.first_bad < (unsigned long long)cnt) {  // reject the batch: nothing applied
      { note_launch(); set_result_k<<<1, 1, 0, st>>>(result, SFK_BAD_OPCODE, (int64_t)s.first_bad, 0, nullptr, 0, 0); }
      return check_launch("set_result");
    }
    // the CU min can reach 0xFFFFFFFF only if some counter climbs that far:
    // counters grow by at most one per insert
    if ((uint64_t)s.cmax + s.ins_before_first_del < 0xFFFFFFFFull)
      return parallel_apply(2, counters, nullptr, nullptr, seeds, nullptr, d, w, 0, 1, ops + t0, ks, cnt, inc_counts, result,
                            workspace, workspace_bytes, st);
    return launch_seq_apply(1, 0, counters, nullptr, nullptr, seeds, nullptr, d, w, 0, 1, ops + t0, ks, nullptr, cnt,
                            inc_counts, result, st);
  });
}

// parallel engine kind per variant (see carve() in sfk_sf.cu); -1: the exact
// one-thread device engine
static int sf_parallel_kind(int variant, int d, int z, int64_t w = 0, int64_t w_prime = 0) {
  if (d > MAXD) return -1;
  if (variant == SFK_VARIANT_SF1) return 1;
  if (variant == SFK_VARIANT_SFF && z >= 1 && z <= 8) return 0;
  if (variant == SFK_VARIANT_SF4 && z >= 1 && z <= 8) return 4;
  if (variant == SFK_VARIANT_SF3 && z >= 1 && z <= 8 && w_prime == (int64_t)z * w) return 5;
  if (variant == SFK_VARIANT_SF2) return 6;
  return -1;
}

static int kind_z(int kind, int z) { return (kind == 0 || kind == 4 || kind == 5) ? z : 1; }

size_t sfk_sf_workspace_size(int variant, int d, int64_t w, int64_t w_prime, int z, int64_t n) {
  const int kind = sf_parallel_kind(variant, d, z, w, w_prime);
  if (kind < 0) return 256;
  // the warp engine takes SFF / SF4 batches up to warp_batch_ops() ops
  // without a workspace (the same test sfk_sf_apply makes; it falls back to
  // the parallel pipeline only for shapes the warp does not fit)
  if ((variant == SFK_VARIANT_SFF || variant == SFK_VARIANT_SF4) && n > 0 && n <= warp_batch_ops() && d <= MAXD &&
      w < (int64_t(1) << 24)) {
    int Z = 1;
    while (Z < z) Z <<= 1;
    if ((int64_t)d * Z <= 32) return 256;
  }
  if ((variant == SFK_VARIANT_SFF || variant == SFK_VARIANT_SF4) && n > warp_batch_ops() && n <= block_batch_ops() &&
      blk_fits(d, w, z, n))
    return 256;  // the block engine needs no workspace
  return parallel_workspace_size(kind, d, w, w_prime, z, std::min<int64_t>(n, chunk_ops(d, kind_z(kind, z))));
}

int sfk_sf_apply(int variant, uint32_t* slim, uint32_t* fat, uint32_t* dsub, const uint64_t* slim_seeds,
                 const uint64_t* fat_seeds, int d, int64_t w, int64_t w_prime, int z, const uint8_t* ops,
                 const void* keys, int key_kind, int rec_len, int64_t n, int64_t* inc_counts, int64_t* result,
                 void* workspace, size_t workspace_bytes, int flags, void* stream) {
  if (check_common(d, w, key_kind, rec_len)) return 1;
  cudaStream_t st = (cudaStream_t)stream;
  const bool flat = variant == SFK_VARIANT_SF1 || variant == SFK_VARIANT_SF2 || variant == SFK_VARIANT_SF3;
  const bool bucketed = variant == SFK_VARIANT_SF4 || variant == SFK_VARIANT_SFF;
  if (!flat && !bucketed) { set_error("unknown SF variant %d", variant); return 1; }
  if (z < 1) { set_error("z must be >= 1"); return 1; }
  if (flat && (w_prime < w || (uint64_t)d * (uint64_t)w_prime >= (1ull << 32))) {
    set_error("bad w_prime=%lld", (long long)w_prime);
    return 1;
  }
  if (bucketed && (uint64_t)d * (uint64_t)w * (uint64_t)z >= (1ull << 32)) { set_error("fat too large"); return 1; }
  if (variant == SFK_VARIANT_SF2 && dsub == nullptr) { set_error("SF2 needs the deletion sub-sketch"); return 1; }
  const int kind = sf_parallel_kind(variant, d, z, w, w_prime);
  KeySrc all{keys, key_kind, rec_len};
  if (bucketed && !(flags & SFK_FLAG_SEQUENTIAL) && n > 0 && n <= warp_batch_ops()) {
    const int rc = launch_seqw_bucket(variant == SFK_VARIANT_SF4 ? 0 : 1, slim, fat, slim_seeds, fat_seeds, d, w, z,
                                      ops, all, n, inc_counts, result, st);
    if (rc >= 0) return rc;
  }
  if (bucketed && !(flags & SFK_FLAG_SEQUENTIAL) && n > warp_batch_ops() && n <= block_batch_ops()) {
    const int rc = launch_blk_bucket(variant == SFK_VARIANT_SF4 ? 0 : 1, slim, fat, slim_seeds, fat_seeds, d, w, z,
                                     ops, all, n, inc_counts, result, st);
    if (rc >= 0) return rc;
  }
  if ((flags & SFK_FLAG_SEQUENTIAL) || kind < 0 || small_batch(n)) {
    if (flat)
      return launch_seq_apply(2, variant, slim, fat, dsub, slim_seeds, fat_seeds, d, w, w_prime, w_prime / w, ops, all,
                              nullptr, n, inc_counts, result, st);
    return launch_seq_apply(3, variant == SFK_VARIANT_SF4 ? 0 : 1, slim, fat, nullptr, slim_seeds, fat_seeds, d, w, 0,
                            z, ops, all, nullptr, n, inc_counts, result, st);
  }
  bool rejected = false;
  if (int r = bad_ops_first(ops, n, chunk_ops(d, kind_z(kind, z)), workspace, workspace_bytes, result, st, &rejected))
    return r;
  if (rejected) return 0;
  return chunked(n, chunk_ops(d, kind_z(kind, z)), result, st, [&](int64_t t0, int64_t cnt) -> int {
    KeySrc ks{key_ptr(keys, key_kind, rec_len, t0), key_kind, rec_len};
    return parallel_apply(kind, slim, fat, dsub, slim_seeds, fat_seeds, d, w, w_prime, z, ops + t0, ks, cnt,
                          inc_counts, result, workspace, workspace_bytes, st);
  });
}

size_t sfk_oracle_workspace_size(int d, int64_t w, int64_t n) {
  if (d > MAXD) return 256;
  return parallel_workspace_size(8, d, w, 0, 1, std::min<int64_t>(n, chunk_ops(d, 1)));
}

int sfk_oracle_slim_apply(uint32_t* slim, const uint64_t* seeds, int d, int64_t w, const void* keys, int key_kind,
                          int rec_len, const int64_t* true_counts, int64_t n, int64_t* inc_counts, int64_t* result,
                          void* workspace, size_t workspace_bytes, int flags, void* stream) {
  if (check_common(d, w, key_kind, rec_len)) return 1;
  cudaStream_t st = (cudaStream_t)stream;
  KeySrc all{keys, key_kind, rec_len};
  bool ok = false;
  if (!(flags & SFK_FLAG_SEQUENTIAL) && d <= MAXD && n > 0 && !small_batch(n))
    if (int r = gated_precheck(true_counts, n, nullptr, nullptr, slim, (int64_t)d * w, workspace, workspace_bytes, &ok, st)) return r;
  if (!ok)
    return launch_seq_apply(4, 0, slim, nullptr, nullptr, seeds, nullptr, d, w, 0, 1, nullptr, all, true_counts, n,
                            inc_counts, result, st);
  return chunked(n, chunk_ops(d, 1), result, st, [&](int64_t t0, int64_t cnt) -> int {
    KeySrc ks{key_ptr(keys, key_kind, rec_len, t0), key_kind, rec_len};
    ExtArgs ext{nullptr, nullptr, 0, 0, true_counts + t0};
    return parallel_apply(8, slim, nullptr, nullptr, seeds, nullptr, d, w, 0, 1, nullptr, ks, cnt, inc_counts, result,
                          workspace, workspace_bytes, st, &ext);
  });
}

// ---------------------------------------------------------------- synthetic streams
int sfk_pcg64_draws(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t offset, int64_t n,
                    const double* cdf, int64_t v, int64_t* ranks, double* uniforms, void* stream) {
  if (offset < 0 || n < 0 || (cdf && (v < 1 || !ranks)) || (!cdf && !uniforms)) {
    set_error("sfk_pcg64_draws: bad arguments");
    return 1;
  }
  return launch_pcg_uniform(state_hi, state_lo, inc_hi, inc_lo, offset, n, cdf, v, ranks, uniforms,
                            (cudaStream_t)stream);
}

size_t sfk_pcg64_bounded_workspace_size(int64_t n, int64_t v) {
  if (n < 0 || v < 1 || v > ((int64_t)1 << 32)) return 256;
  return pcg_bounded_workspace_size(n, v);
}

int sfk_pcg64_bounded(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t offset64,
                      int64_t n, int64_t v, int64_t* out, int64_t* next_offset64, void* workspace,
                      size_t workspace_bytes, void* stream) {
  if (n < 0 || v < 1 || v > ((int64_t)1 << 32) || !next_offset64) {
    set_error("sfk_pcg64_bounded: bad arguments (1 <= v <= 2^32)");
    return 1;
  }
  return launch_pcg_bounded(state_hi, state_lo, inc_hi, inc_lo, offset64, n, v, out, next_offset64, workspace,
                            workspace_bytes, (cudaStream_t)stream);
}

size_t sfk_interleave_workspace_size(int64_t v) { return (size_t)(v > 0 ? v : 1) * 3 * 8 + 3 * 256; }

int sfk_interleave_deletions(const int64_t* candidates, const double* decide, const double* pick, double p,
                             int64_t n, int64_t v, uint8_t* ops, int64_t* ranks, void* workspace,
                             size_t workspace_bytes, void* stream) {
  if (n < 0 || v < 1) { set_error("sfk_interleave_deletions: bad sizes"); return 1; }
  return launch_interleave(candidates, decide, pick, p, n, v, ops, ranks, workspace, workspace_bytes,
                           (cudaStream_t)stream);
}

// ---------------------------------------------------------------- trace ingestion
size_t sfk_trace_workspace_size(int64_t nbytes) { return trace_workspace_size(nbytes); }

int sfk_trace_parse_lines(const uint8_t* text, int64_t nbytes, int64_t* line_pos, uint8_t* status, uint8_t* op,
                          uint64_t* key, int64_t* info, void* workspace, size_t workspace_bytes, void* stream) {
  if (nbytes < 0) { set_error("negative trace size"); return 1; }
  return trace_parse_lines(text, nbytes, line_pos, status, op, key, info, workspace, workspace_bytes,
                           (cudaStream_t)stream);
}

int sfk_trace_compact(const uint8_t* status, const uint8_t* op, const uint64_t* key, int64_t nlines, uint8_t* ops,
                      uint64_t* keys, int64_t* n_out, void* workspace, size_t workspace_bytes, int64_t nbytes,
                      void* stream) {
  return trace_compact(status, op, key, nlines, ops, keys, n_out, workspace, workspace_bytes, nbytes,
                       (cudaStream_t)stream);
}

// ---------------------------------------------------------------- Count / CML
size_t sfk_count_workspace_size(int d, int64_t w, int64_t n) { return 4096; }

int sfk_count_apply(int32_t* counters, const uint64_t* seeds, int d, int64_t w, const uint8_t* ops, const void* keys,
                    int key_kind, int rec_len, int64_t n, int64_t* result, void* workspace, size_t workspace_bytes,
                    int flags, void* stream) {
  if (check_common(d, w, key_kind, rec_len)) return 1;
  cudaStream_t st = (cudaStream_t)stream;
  KeySrc all{keys, key_kind, rec_len};
  if ((flags & SFK_FLAG_SEQUENTIAL) || d > MAXD || small_batch(n))
    return launch_seq_ext(5, counters, seeds, d, w, ops, all, n, nullptr, 0, 0, result, st);
  return chunked(n, chunk_ops(d, 1), result, st, [&](int64_t t0, int64_t cnt) -> int {
    KeySrc ks{key_ptr(keys, key_kind, rec_len, t0), key_kind, rec_len};
    Stats s;
    if (int r = collect_stats(ops + t0, cnt, reinterpret_cast<const uint32_t*>(counters), (int64_t)d * w, workspace,
                              workspace_bytes, &s, st, 0x80000000u))
      return r;
    // every counter moves by at most one per op: no op can meet a bound
    const int64_t cmax = (int64_t)(int32_t)(s.cmax ^ 0x80000000u), cmin = (int64_t)(int32_t)(s.cmin ^ 0x80000000u);
    if (cmax + cnt <= 2147483647ll && cmin - cnt >= -2147483648ll) {
      if (int r = count_fast(counters, seeds, d, w, ops + t0, ks, cnt, st)) return r;
      { note_launch(); set_result_k<<<1, 1, 0, st>>>(result, SFK_OK, -1, (int64_t)s.n_ins, nullptr, 0, 0); }
      return check_launch("set_result");
    }
    return launch_seq_ext(5, counters, seeds, d, w, ops + t0, ks, cnt, nullptr, 0, 0, result, st);
  });
}

int sfk_count_query(const int32_t* counters, const uint64_t* seeds, int d, int64_t w, const void* keys, int key_kind,
                    int rec_len, int64_t n, int64_t* out, void* stream) {
  if (check_common(d, w, key_kind, rec_len)) return 1;
  return ext_query(0, counters, seeds, d, w, KeySrc{keys, key_kind, rec_len}, n, nullptr, out, (cudaStream_t)stream);
}

size_t sfk_cml_workspace_size(int d, int64_t w, int64_t n) {
  if (d > MAXD) return 256;
  return parallel_workspace_size(7, d, w, 0, 1, std::min<int64_t>(n, chunk_ops(d, 1)));
}

int sfk_cml_apply(uint16_t* exps, const uint64_t* seeds, int d, int64_t w, const uint8_t* ops, const void* keys,
                  int key_kind, int rec_len, int64_t n, const double* gate, uint64_t rng_seed, int64_t start_pos,
                  int64_t* result, void* workspace, size_t workspace_bytes, int flags, void* stream) {
  if (check_common(d, w, key_kind, rec_len)) return 1;
  if (gate == nullptr) { set_error("CML apply needs the gate table"); return 1; }
  cudaStream_t st = (cudaStream_t)stream;
  KeySrc all{keys, key_kind, rec_len};
  bool ok = false;
  if (!(flags & SFK_FLAG_SEQUENTIAL) && d <= MAXD && n > 0 && !small_batch(n))
    if (int r = gated_precheck(nullptr, n, gate, exps, nullptr, (int64_t)d * w, workspace, workspace_bytes, &ok, st)) return r;
  if (!ok) return launch_seq_ext(6, exps, seeds, d, w, ops, all, n, gate, rng_seed, start_pos, result, st);
  return chunked(n, chunk_ops(d, 1), result, st, [&](int64_t t0, int64_t cnt) -> int {
    KeySrc ks{key_ptr(keys, key_kind, rec_len, t0), key_kind, rec_len};
    // every op before this chunk was an insert (a failing chunk ends the batch)
    ExtArgs ext{exps, gate, rng_seed, start_pos + t0, nullptr};
    return parallel_apply(7, nullptr, nullptr, nullptr, seeds, nullptr, d, w, 0, 1, ops + t0, ks, cnt, nullptr, result,
                          workspace, workspace_bytes, st, &ext);
  });
}

int sfk_cml_query(const uint16_t* exps, const uint64_t* seeds, int d, int64_t w, const void* keys, int key_kind,
                  int rec_len, int64_t n, const int64_t* value_table, int64_t* out, void* stream) {
  if (check_common(d, w, key_kind, rec_len)) return 1;
  return ext_query(1, exps, seeds, d, w, KeySrc{keys, key_kind, rec_len}, n, value_table, out, (cudaStream_t)stream);
}

}  // extern "C"
