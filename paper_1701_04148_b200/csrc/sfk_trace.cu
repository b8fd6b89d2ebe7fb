// Trace ingestion on the GPU (workloads.read_trace / load_trace,
// workloads.py:132-172): the text of an "OP,key" trace is parsed where the
// sketches consume it. One pass flags line starts (Python's universal
// newlines: \n, \r\n and a lone \r all end a line), a select compacts them,
// one thread per line applies the reference's rules (str.strip, '#'
// comments, split(",") into exactly two parts, op token I / D, int(key, 10)
// with sign and digit-group underscores, 64-bit range), and a scan compacts
// the op lines into (ops, keys).
//
// Per line status: 0 skipped (blank / comment), 1 op, 2 "expected 'OP,key'",
// 3 unknown op token, 4 bad key, 5 key out of 64-bit range, 6 non-ASCII bytes
// (Python's Unicode whitespace and digit rules: the host finishes those
// lines). The host formats the first error's message from its line text.
#include <cub/cub.cuh>

#include "sfk_common.cuh"

namespace sfk {

int sm_count();

enum : uint8_t { TL_SKIP = 0, TL_OP = 1, TL_SPLIT = 2, TL_TOKEN = 3, TL_KEY = 4, TL_RANGE = 5, TL_COMPLEX = 6 };

__global__ void trace_starts_k(const uint8_t* __restrict__ txt, int64_t nb, uint8_t* __restrict__ flag) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nb; i += (int64_t)gridDim.x * blockDim.x) {
    bool s = i == 0;
    if (!s) {
      const uint8_t p = txt[i - 1];
      s = p == '\n' || (p == '\r' && txt[i] != '\n');
    }
    flag[i] = s ? 1 : 0;
  }
}

// Python str.isspace() on ASCII: \t \n \v \f \r, \x1c-\x1f, space
__device__ __forceinline__ bool py_space(uint8_t c) { return (c >= 9 && c <= 13) || (c >= 28 && c <= 32); }

// int(text, 10) on ASCII text already stripped: [+-] digit (_? digit)*
__device__ __forceinline__ uint8_t parse_key(const uint8_t* t, int64_t a, int64_t b, uint64_t* out) {
  if (a >= b) return TL_KEY;
  bool neg = false;
  if (t[a] == '+' || t[a] == '-') {
    neg = t[a] == '-';
    ++a;
  }
  if (a >= b) return TL_KEY;
  unsigned long long v = 0;
  bool big = false, prev_digit = false;
  for (int64_t i = a; i < b; ++i) {
    const uint8_t c = t[i];
    if (c >= '0' && c <= '9') {
      const unsigned long long d = c - '0';
      if (!big) {
        if (v > (0xFFFFFFFFFFFFFFFFull - d) / 10ull) big = true;
        else v = v * 10ull + d;
      }
      prev_digit = true;
    } else if (c == '_' && prev_digit && i + 1 < b && t[i + 1] >= '0' && t[i + 1] <= '9') {
      prev_digit = false;
    } else {
      return TL_KEY;
    }
  }
  if (big || (neg && v != 0)) return TL_RANGE;
  *out = v;
  return TL_OP;
}

__global__ void trace_lines_k(const uint8_t* __restrict__ txt, int64_t nb, const int64_t* __restrict__ pos,
                              const int64_t* __restrict__ nlines_p, uint8_t* __restrict__ status,
                              uint8_t* __restrict__ lop, uint64_t* __restrict__ lkey) {
  const int64_t nl = *nlines_p;
  for (int64_t L = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; L < nl; L += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = pos[L], b = L + 1 < nl ? pos[L + 1] : nb;
    uint8_t st = TL_SKIP, op = 0;
    uint64_t key = 0;
    bool ascii = true;
    for (int64_t i = a; i < b; ++i) ascii = ascii && txt[i] < 0x80;
    if (!ascii) {
      st = TL_COMPLEX;
    } else {
      while (a < b && py_space(txt[a])) ++a;
      while (b > a && py_space(txt[b - 1])) --b;
      if (a < b && txt[a] != '#') {
        int64_t comma = -1;
        int commas = 0;
        for (int64_t i = a; i < b; ++i)
          if (txt[i] == ',') {
            ++commas;
            comma = i;
          }
        if (commas != 1) {
          st = TL_SPLIT;
        } else {
          int64_t ta = a, tb = comma, ka = comma + 1, kb = b;
          while (ta < tb && py_space(txt[ta])) ++ta;
          while (tb > ta && py_space(txt[tb - 1])) --tb;
          while (ka < kb && py_space(txt[ka])) ++ka;
          while (kb > ka && py_space(txt[kb - 1])) --kb;
          if (tb - ta != 1 || (txt[ta] != 'I' && txt[ta] != 'D')) {
            st = TL_TOKEN;
          } else {
            op = txt[ta] == 'I' ? 0 : 1;
            st = parse_key(txt, ka, kb, &key);
          }
        }
      }
    }
    status[L] = st;
    lop[L] = op;
    lkey[L] = key;
  }
}

__global__ void trace_opflag_k(const uint8_t* __restrict__ status, const int64_t* __restrict__ nlines_p,
                               uint32_t* __restrict__ isop, unsigned long long* __restrict__ summary) {
  // summary: [0] first error line (or ~0), [1] complex lines
  const int64_t nl = *nlines_p;
  for (int64_t L = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; L < nl; L += (int64_t)gridDim.x * blockDim.x) {
    const uint8_t st = status[L];
    isop[L] = st == TL_OP ? 1u : 0u;
    if (st >= TL_SPLIT && st <= TL_RANGE) atomicMin(summary, (unsigned long long)L);
    if (st == TL_COMPLEX) atomicAdd(summary + 1, 1ull);
  }
}

__global__ void trace_scatter_k(const uint8_t* __restrict__ status, const uint8_t* __restrict__ lop,
                                const uint64_t* __restrict__ lkey, const uint32_t* __restrict__ opos,
                                const int64_t* __restrict__ nlines_p, uint8_t* __restrict__ ops,
                                uint64_t* __restrict__ keys) {
  const int64_t nl = *nlines_p;
  for (int64_t L = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; L < nl; L += (int64_t)gridDim.x * blockDim.x) {
    if (status[L] != TL_OP) continue;
    ops[opos[L]] = lop[L];
    keys[opos[L]] = lkey[L];
  }
}

struct TraceWs {
  uint8_t* flag;
  int64_t* pos;
  int64_t* nlines;
  unsigned long long* summary;
  uint32_t* isop;
  uint32_t* opos;
  void* tmp;
  size_t tmp_bytes;
  size_t total;
  bool ok;
};

static size_t trace_tmp_bytes(int64_t nb) {
  size_t a = 0, b = 0;
  cub::DeviceSelect::Flagged(nullptr, a, cub::CountingInputIterator<int64_t>(0), (const uint8_t*)nullptr,
                             (int64_t*)nullptr, (int64_t*)nullptr, (int64_t)nb);
  cub::DeviceScan::ExclusiveSum(nullptr, b, (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)std::min<int64_t>(nb, 1 << 30));
  return std::max(a, b);
}

static TraceWs trace_carve(void* base, size_t cap, int64_t nb) {
  Carver cv(base, cap);
  TraceWs w{};
  const uint64_t n = (uint64_t)(nb > 0 ? nb : 1);
  w.flag = cv.take<uint8_t>(n);
  w.pos = cv.take<int64_t>(n + 1);
  w.nlines = cv.take<int64_t>(1);
  w.summary = cv.take<unsigned long long>(2);
  w.isop = cv.take<uint32_t>(n + 1);
  w.opos = cv.take<uint32_t>(n + 1);
  w.tmp_bytes = trace_tmp_bytes((int64_t)n + 1);
  w.tmp = cv.take<char>(w.tmp_bytes);
  w.total = cv.off + 256;
  w.ok = cv.ok;
  return w;
}

size_t trace_workspace_size(int64_t nb) { return trace_carve(nullptr, ~size_t(0), nb).total; }

static int64_t tgrid(int64_t n) {
  const int64_t cap = (int64_t)sm_count() * 16;
  int64_t g = (n + 255) / 256;
  return g < 1 ? 1 : (g > cap ? cap : g);
}

// Phase 1: per-line status / op / key (line arrays are caller-provided,
// nb + 1 entries each); out_info (host) = {lines, first error line or -1,
// complex lines}.
int trace_parse_lines(const uint8_t* txt, int64_t nb, int64_t* line_pos, uint8_t* status, uint8_t* lop, uint64_t* lkey,
                      int64_t* out_info, void* ws, size_t ws_bytes, cudaStream_t st) {
  TraceWs w = trace_carve(ws, ws_bytes, nb);
  if (!w.ok || ws == nullptr) {
    set_error("trace workspace too small: need %zu bytes, got %zu", w.total, ws_bytes);
    return 1;
  }
  cudaMemsetAsync(w.nlines, 0, 8, st);
  cudaMemsetAsync(w.summary, 0xFF, 8, st);
  cudaMemsetAsync(w.summary + 1, 0, 8, st);
  if (nb > 0) {
    { note_launch(); trace_starts_k<<<tgrid(nb), 256, 0, st>>>(txt, nb, w.flag); }
    size_t bytes = w.tmp_bytes;
    cudaError_t e = cub::DeviceSelect::Flagged(w.tmp, bytes, cub::CountingInputIterator<int64_t>(0), w.flag, line_pos,
                                               w.nlines, nb, st);
    if (e != cudaSuccess) { set_error("trace select: %s", cudaGetErrorString(e)); return (int)e; }
    { note_launch(); trace_lines_k<<<tgrid(nb / 8 + 1), 256, 0, st>>>(txt, nb, line_pos, w.nlines, status, lop, lkey); }
    { note_launch(); trace_opflag_k<<<tgrid(nb / 8 + 1), 256, 0, st>>>(status, w.nlines, w.isop, w.summary); }
  }
  if (int r = check_launch("trace_parse")) return r;
  int64_t h[3];
  cudaMemcpyAsync(&h[0], w.nlines, 8, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&h[1], w.summary, 16, cudaMemcpyDeviceToHost, st);
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) { set_error("trace sync: %s", cudaGetErrorString(e)); return (int)e; }
  out_info[0] = h[0];
  out_info[1] = (uint64_t)h[1] == ~0ull ? -1 : h[1];
  out_info[2] = h[2];
  return 0;
}

// Phase 2: compact the op lines (status 1) into ops / keys; returns the count.
int trace_compact(const uint8_t* status, const uint8_t* lop, const uint64_t* lkey, int64_t nlines, uint8_t* ops,
                  uint64_t* keys, int64_t* out_n, void* ws, size_t ws_bytes, int64_t nb, cudaStream_t st) {
  TraceWs w = trace_carve(ws, ws_bytes, nb);
  if (!w.ok || ws == nullptr) {
    set_error("trace workspace too small: need %zu bytes, got %zu", w.total, ws_bytes);
    return 1;
  }
  if (nlines <= 0) { *out_n = 0; return 0; }
  if (nlines >= (int64_t)1 << 31) { set_error("trace: too many lines"); return 1; }
  cudaMemcpyAsync(w.nlines, &nlines, 8, cudaMemcpyHostToDevice, st);
  cudaMemsetAsync(w.summary, 0xFF, 8, st);
  { note_launch(); trace_opflag_k<<<tgrid(nlines), 256, 0, st>>>(status, w.nlines, w.isop, w.summary); }
  cudaMemsetAsync(w.isop + nlines, 0, 4, st);
  size_t bytes = w.tmp_bytes;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(w.tmp, bytes, w.isop, w.opos, (int)(nlines + 1), st);
  if (e != cudaSuccess) { set_error("trace scan: %s", cudaGetErrorString(e)); return (int)e; }
  { note_launch(); trace_scatter_k<<<tgrid(nlines), 256, 0, st>>>(status, lop, lkey, w.opos, w.nlines, ops, keys); }
  if (int r = check_launch("trace_compact")) return r;
  uint32_t cnt = 0;
  cudaMemcpyAsync(&cnt, w.opos + nlines, 4, cudaMemcpyDeviceToHost, st);
  e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) { set_error("trace sync: %s", cudaGetErrorString(e)); return (int)e; }
  *out_n = cnt;
  return 0;
}

}  // namespace sfk
