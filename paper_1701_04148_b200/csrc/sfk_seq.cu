// Exact sequential device engine: one thread replays a batch in stream order
// with the reference's per-op rules (_kernels.py:62-115, 244-411).
//
// It is the GPU path for the configurations the parallel engines do not
// cover (SF2/SF3/SF4 variants, d > 8, CU batches that could saturate, the
// oracle-assisted mode) and the cross-check the parity tests run against the
// parallel engines (flag SFK_FLAG_SEQUENTIAL). It is slow (one L2 round trip
// per counter touch) but bit-exact by construction.
#include "sfk_common.cuh"

namespace sfk {

struct SeqArgs {
  uint32_t* slim;  // counters for CM/CU
  uint32_t* fat;
  uint32_t* dsub;
  Seeds<MAXSEEDS> s_seeds;  // slim / bucket / CM seeds
  Seeds<MAXSEEDS> f_seeds;  // fat / slot seeds
  int d;
  int64_t w, wp, z;
  Mod wm, wpm, zm;
  const uint8_t* ops;
  KeySrc keys;
  const int64_t* true_counts;
  uint16_t* exps;        // CML exponents
  const double* gate;    // CML: gate[c] = base ** -c (libm pow, computed by the caller)
  uint64_t rng_seed;     // CML coin-flip stream
  int64_t start_pos;     // CML: inserts the sketch saw before this batch
  int64_t n;
  int64_t* inc;
  int64_t* result;
};

// kind: 0 CM, 1 CU, 2 SF flat (variant 1/2/3), 3 SF bucketed (mode 0/1/2), 4 oracle-assisted slim,
//       5 Count (signed int32 counters), 6 CML (u16 exponents)
__global__ void seq_apply_k(SeqArgs a, int kind, int variant) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int d = a.d;
  int64_t idx[MAXSEEDS], idx2[MAXSEEDS];
  int64_t n_ins = 0;
  int64_t status = SFK_OK, bad = -1;
  const int64_t w = a.w, wp = a.wp, z = a.z;
  if (a.ops) {  // a bad op code rejects the whole batch before anything is applied
    for (int64_t t = 0; t < a.n; ++t)
      if (a.ops[t] > 1) {
        a.result[0] = SFK_BAD_OPCODE;
        a.result[1] = t;
        a.result[2] = 0;
        return;
      }
  }
  for (int64_t t = 0; t < a.n; ++t) {
    const uint64_t key = load_key(a.keys, t);
    const int op = a.ops ? a.ops[t] : 0;
    if (kind == 5) {  // count_apply, _kernels.py:118-146
      int32_t* c = reinterpret_cast<int32_t*>(a.slim);
      int dl[MAXSEEDS];
      bool fail = false;
      for (int i = 0; i < d; ++i) {
        idx[i] = (int64_t)bucket(key, a.s_seeds.s[i], a.wm);
        int s = (mix64(key ^ a.s_seeds.s[i] ^ 0xA5A5A5A5A5A5A5A5ull) & 1ull) ? -1 : 1;
        if (op) s = -s;
        const int32_t v = c[i * w + idx[i]];
        if ((s > 0 && v == 2147483647) || (s < 0 && v == (-2147483647 - 1))) fail = true;
        dl[i] = s;
      }
      if (fail) { status = SFK_SATURATED; bad = t; break; }
      for (int i = 0; i < d; ++i) c[i * w + idx[i]] += dl[i];
      if (op == 0) ++n_ins;
    } else if (kind == 6) {  // cml_apply, _kernels.py:182-211
      if (op != 0) { status = SFK_UNSUPPORTED; bad = t; break; }
      uint32_t cmin = 0xFFFFu;
      for (int i = 0; i < d; ++i) {
        idx[i] = (int64_t)bucket(key, a.s_seeds.s[i], a.wm);
        cmin = min(cmin, (uint32_t)a.exps[i * w + idx[i]]);
      }
      const uint64_t pos = (uint64_t)(a.start_pos + n_ins);
      const uint64_t u = mix64(a.rng_seed + (pos + 1ull) * 0x9E3779B97F4A7C15ull);
      const double uf = (double)(u >> 11) * (1.0 / 9007199254740992.0);
      if (uf < a.gate[cmin]) {
        if (cmin == 0xFFFFu) { status = SFK_SATURATED; bad = t; break; }
        for (int i = 0; i < d; ++i)
          if (a.exps[i * w + idx[i]] == cmin) a.exps[i * w + idx[i]] += 1;
      }
      ++n_ins;
    } else if (kind == 0) {  // cm_apply, _kernels.py:62-88
      bool fail = false;
      for (int i = 0; i < d; ++i) {
        idx[i] = (int64_t)bucket(key, a.s_seeds.s[i], a.wm);
        uint32_t v = a.slim[i * w + idx[i]];
        if (op == 0 ? v == U32MAX : v == 0u) fail = true;
      }
      if (fail) { status = op == 0 ? SFK_SATURATED : SFK_PHANTOM; bad = t; break; }
      for (int i = 0; i < d; ++i) {
        if (op == 0) { a.slim[i * w + idx[i]] += 1u; a.inc[i] += 1; }
        else a.slim[i * w + idx[i]] -= 1u;
      }
      if (op == 0) ++n_ins;
    } else if (kind == 1 || kind == 4) {  // cu_apply 91-115, oracle_slim_apply 387-411
      if (kind == 1 && op != 0) { status = SFK_UNSUPPORTED; bad = t; break; }
      uint64_t m = U64MAX;
      for (int i = 0; i < d; ++i) {
        idx[i] = (int64_t)bucket(key, a.s_seeds.s[i], a.wm);
        uint64_t v = a.slim[i * w + idx[i]];
        if (v < m) m = v;
      }
      bool raise = true;
      if (kind == 4) raise = m < (uint64_t)a.true_counts[t];
      if (raise) {
        if (m >= 0xFFFFFFFFull) { status = SFK_SATURATED; bad = t; break; }
        for (int i = 0; i < d; ++i)
          if ((uint64_t)a.slim[i * w + idx[i]] == m) { a.slim[i * w + idx[i]] += 1u; a.inc[i] += 1; }
      }
      ++n_ins;
    } else if (kind == 2) {  // sf_flat_apply 244-315
      int64_t* sidx = idx;
      int64_t* fidx = idx2;
      for (int i = 0; i < d; ++i) {
        if (variant == 3) {
          uint64_t g = bucket(key, a.f_seeds.s[i], a.wpm);
          fidx[i] = (int64_t)g;
          sidx[i] = (int64_t)fmod64(g, a.wm);
        } else {
          fidx[i] = (int64_t)bucket(key, a.f_seeds.s[i], a.wpm);
          sidx[i] = (int64_t)bucket(key, a.s_seeds.s[i], a.wm);
        }
      }
      if (op == 0) {
        bool fail = false;
        for (int i = 0; i < d; ++i) {
          if (a.fat[i * wp + fidx[i]] == U32MAX) fail = true;
          if (variant == 2 && a.dsub[i * w + sidx[i]] == U32MAX) fail = true;
        }
        if (fail) { status = SFK_SATURATED; bad = t; break; }
        uint64_t bmin = U64MAX;
        for (int i = 0; i < d; ++i) {
          a.fat[i * wp + fidx[i]] += 1u;
          uint64_t v = a.fat[i * wp + fidx[i]];
          if (v < bmin) bmin = v;
          if (variant == 2) a.dsub[i * w + sidx[i]] += 1u;
        }
        uint64_t m = U64MAX;
        for (int i = 0; i < d; ++i) {
          uint64_t v = a.slim[i * w + sidx[i]];
          if (v < m) m = v;
        }
        if (m < bmin)
          for (int i = 0; i < d; ++i)
            if ((uint64_t)a.slim[i * w + sidx[i]] == m) { a.slim[i * w + sidx[i]] += 1u; a.inc[i] += 1; }
        ++n_ins;
      } else {
        if (variant == 1) { status = SFK_UNSUPPORTED; bad = t; break; }
        bool fail = false;
        for (int i = 0; i < d; ++i) {
          if (a.fat[i * wp + fidx[i]] == 0u) fail = true;
          if (variant == 2 && a.dsub[i * w + sidx[i]] == 0u) fail = true;
        }
        if (fail) { status = SFK_PHANTOM; bad = t; break; }
        for (int i = 0; i < d; ++i) {
          a.fat[i * wp + fidx[i]] -= 1u;
          uint32_t* sc = &a.slim[i * w + sidx[i]];
          if (variant == 2) {
            a.dsub[i * w + sidx[i]] -= 1u;
            if (*sc > a.dsub[i * w + sidx[i]]) *sc -= 1u;
          } else {
            uint64_t total = 0;
            for (int64_t m2 = 0; m2 < z; ++m2) total += a.fat[i * wp + sidx[i] + m2 * w];
            if ((uint64_t)*sc > total) *sc -= 1u;
          }
        }
      }
    } else {  // kind 3: sf_bucket_apply 318-384
      int64_t* jidx = idx;
      int64_t* kidx = idx2;
      for (int i = 0; i < d; ++i) {
        jidx[i] = (int64_t)bucket(key, a.s_seeds.s[i], a.wm);
        kidx[i] = (int64_t)bucket(key, a.f_seeds.s[i], a.zm);
      }
#define FATC(i, j, k) a.fat[((int64_t)(i) * w + (j)) * z + (k)]
      if (op == 0) {
        bool fail = false;
        for (int i = 0; i < d; ++i)
          if (FATC(i, jidx[i], kidx[i]) == U32MAX) fail = true;
        if (fail) { status = SFK_SATURATED; bad = t; break; }
        uint64_t bmin = U64MAX;
        for (int i = 0; i < d; ++i) {
          FATC(i, jidx[i], kidx[i]) += 1u;
          uint64_t v = FATC(i, jidx[i], kidx[i]);
          if (v < bmin) bmin = v;
        }
        uint64_t m = U64MAX;
        for (int i = 0; i < d; ++i) {
          uint64_t v = a.slim[i * w + jidx[i]];
          if (v < m) m = v;
        }
        if (m < bmin)
          for (int i = 0; i < d; ++i)
            if ((uint64_t)a.slim[i * w + jidx[i]] == m) { a.slim[i * w + jidx[i]] += 1u; a.inc[i] += 1; }
        ++n_ins;
      } else {
        bool fail = false;
        for (int i = 0; i < d; ++i)
          if (FATC(i, jidx[i], kidx[i]) == 0u) fail = true;
        if (fail) { status = SFK_PHANTOM; bad = t; break; }
        for (int i = 0; i < d; ++i) {
          const int64_t j = jidx[i];
          uint32_t pre = 0;
          if (variant == 2)
            for (int64_t k = 0; k < z; ++k) pre = max(pre, FATC(i, j, k));
          FATC(i, j, kidx[i]) -= 1u;
          uint32_t* sc = &a.slim[i * w + j];
          if (variant == 0) {
            uint64_t total = 0;
            for (int64_t k = 0; k < z; ++k) total += FATC(i, j, k);
            if ((uint64_t)*sc > total) *sc -= 1u;
          } else {
            uint32_t mx = 0;
            for (int64_t k = 0; k < z; ++k) mx = max(mx, FATC(i, j, k));
            if (variant == 1) {
              if (*sc > mx) *sc = mx;
            } else if (mx != pre && *sc > mx) {
              *sc = mx;
            }
          }
        }
      }
#undef FATC
    }
  }
  a.result[0] = status;
  a.result[1] = bad;
  a.result[2] = n_ins;
}

// Warp-cooperative exact engine for small SFF / SF4 batches
// (sf_bucket_apply, _kernels.py:318-384). Ops still run one after another,
// but lane (i, k) owns fat slot k of row i's bucket (and lane (i, 0) the slim
// cell): the d x z counter reads of an op are one round of parallel loads, the
// "all rows first" failure checks are a ballot, and the minima / row maxima /
// row sums are warp reductions. A lane always handles the same (row, slot)
// position, so the only cross-op dependencies through memory are the lane's
// own earlier stores (program order). The next P ops are hashed ahead and
// their counter lines prefetched into L1. Z = z rounded up to a power of two
// (row groups are aligned lane segments), d * Z <= 32.
template <int Z>
__global__ void __launch_bounds__(32) seqw_bucket_k(SeqArgs a, int variant) {
  constexpr int P = 8;
  const int lane = threadIdx.x;
  {  // a bad op code rejects the whole batch before anything is applied
    unsigned long long fb = ~0ull;
    for (int64_t t = lane; t < a.n; t += 32)
      if (a.ops[t] > 1) {
        fb = (unsigned long long)t;
        break;
      }
    for (int o = 16; o > 0; o >>= 1) fb = min(fb, __shfl_xor_sync(0xFFFFFFFFu, fb, o));
    if (fb != ~0ull) {
      if (lane == 0) {
        a.result[0] = SFK_BAD_OPCODE;
        a.result[1] = (int64_t)fb;
        a.result[2] = 0;
      }
      return;
    }
  }
  const int i = lane / Z, k = lane % Z;
  const bool act = i < a.d && k < (int)a.z;
  const int64_t w = a.w, z = a.z, n = a.n;
  uint32_t* fat_row = a.fat + (int64_t)(act ? i : 0) * w * z;
  uint32_t* slim_row = a.slim + (int64_t)(act ? i : 0) * w;
  // Ops arrive 32 at a time: lane l holds op base + l and hashes it for
  // every row (independent chains, good ILP; a single dependent hash per op
  // and row would leave the warp latency-bound); op t's row-i bucket and slot
  // are then d shuffles away. The next block is hashed one block ahead.
  // code = bucket | slot << 24 (w < 2^24, z <= 32)
  uint32_t hcur[MAXD], hnext[MAXD];
  uint32_t ocur = 0, onext = 0;
  auto hash_block = [&](int64_t b0, uint32_t (&h)[MAXD], uint32_t& o) {
    const int64_t t = b0 + lane;
    o = 0;
#pragma unroll
    for (int r = 0; r < MAXD; ++r) h[r] = 0;
    if (t >= n) return;
    const uint64_t key = load_key(a.keys, t);
    o = a.ops[t];
#pragma unroll
    for (int r = 0; r < MAXD; ++r)
      if (r < a.d)
        h[r] = (uint32_t)bucket(key, a.s_seeds.s[r], a.wm) | ((uint32_t)bucket(key, a.f_seeds.s[r], a.zm) << 24);
  };
  hash_block(0, hcur, ocur);
  hash_block(32, hnext, onext);
  // this lane's (row i) code for op base + q, q < 64
  auto code_of = [&](int q) -> uint32_t {
    uint32_t c = 0;
#pragma unroll
    for (int r = 0; r < MAXD; ++r) {
      if (r >= a.d) break;
      const uint32_t v = q < 32 ? __shfl_sync(0xFFFFFFFFu, hcur[r], q & 31) : __shfl_sync(0xFFFFFFFFu, hnext[r], q & 31);
      if (r == i) c = v;
    }
    return c;
  };
  // ring of the next P ops: this lane's bucket code and its fat word / slim
  // word for that op, loaded P ops ahead. The loads were issued before the
  // ops in between were applied, so every store forwards its value into the
  // ring entries of the same cell (a lane always handles the same (row,
  // slot), so forwarding is lane-local).
  uint32_t rc[P], rf[P], rs[P];
  auto fetch_op = [&](int64_t t, int q, uint32_t& c, uint32_t& fv, uint32_t& sv) {
    c = code_of(q);
    fv = 0;
    sv = 0;
    if (!act || t >= n) {
      c = 0xFFFFFFFFu;
      return;
    }
    const uint32_t j = c & 0xFFFFFFu;
    fv = fat_row[(int64_t)j * z + k];
    if (k == 0) sv = slim_row[j];
  };
#pragma unroll
  for (int q = 0; q < P; ++q) fetch_op(q, q, rc[q], rf[q], rs[q]);
  int64_t n_ins = 0, status = SFK_OK, bad = -1;
  int64_t incl = 0;
  for (int64_t base = 0; base < n && status == SFK_OK; base += 32) {
    const int cnt = (int)min((int64_t)32, n - base);
    for (int q = 0; q < cnt; ++q) {
      const int64_t t = base + q;
      const uint32_t c = rc[0];
      uint32_t fv = rf[0], sv = rs[0];
#pragma unroll
      for (int r = 0; r < P - 1; ++r) rc[r] = rc[r + 1], rf[r] = rf[r + 1], rs[r] = rs[r + 1];
      fetch_op(t + P, q + P, rc[P - 1], rf[P - 1], rs[P - 1]);  // loads in flight for P ops
      const int op = (int)__shfl_sync(0xFFFFFFFFu, ocur, q);
      const uint32_t j = c & 0xFFFFFFu, kk = c >> 24;
      uint32_t* fp = fat_row + (int64_t)j * z + k;
      uint32_t* sp = slim_row + j;
      const bool own = act && (uint32_t)k == kk;
      const uint32_t fv0 = fv, sv0 = sv;
      if (op == 0) {
        if (__any_sync(0xFFFFFFFFu, own && fv == U32MAX)) { status = SFK_SATURATED; bad = t; break; }
        if (own) ++fv;
        const uint32_t bmin = __reduce_min_sync(0xFFFFFFFFu, own ? fv : U32MAX);
        const uint32_t m = __reduce_min_sync(0xFFFFFFFFu, (act && k == 0) ? sv : U32MAX);
        if (act && k == 0 && m < bmin && sv == m) {
          ++sv;
          ++incl;
        }
        ++n_ins;
      } else {
        if (__any_sync(0xFFFFFFFFu, own && fv == 0u)) { status = SFK_PHANTOM; bad = t; break; }
        if (own) --fv;
        if (variant == 1) {  // SFF: clamp the slim cell to the bucket's maximum
          uint32_t mx = act ? fv : 0u;
#pragma unroll
          for (int o = 1; o < Z; o <<= 1) mx = max(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
          if (act && k == 0 && sv > mx) sv = mx;
        } else {  // SF4: decrement when above the bucket's sum
          unsigned long long sum = act ? fv : 0u;
#pragma unroll
          for (int o = 1; o < Z; o <<= 1) sum += __shfl_xor_sync(0xFFFFFFFFu, sum, o);
          if (act && k == 0 && (unsigned long long)sv > sum) sv -= 1u;
        }
      }
      if (act) {
        if (fv != fv0) *fp = fv;
        if (k == 0 && sv != sv0) *sp = sv;
        // forward into the ring: the same bucket of this row, for the later ops
#pragma unroll
        for (int r = 0; r < P; ++r)
          if ((rc[r] & 0xFFFFFFu) == j) rf[r] = fv, rs[r] = sv;
      }
    }
    // slide the block window
#pragma unroll
    for (int r = 0; r < MAXD; ++r) hcur[r] = hnext[r];
    ocur = onext;
    hash_block(base + 64, hnext, onext);
  }
  if (act && k == 0 && incl) atomicAdd(reinterpret_cast<unsigned long long*>(a.inc + i), (unsigned long long)incl);
  if (lane == 0) {
    a.result[0] = status;
    a.result[1] = bad;
    a.result[2] = n_ins;
  }
}

// the warp engine for an SFF (variant 1) / SF4 (variant 0) batch, or -1 if
// the shape does not fit one warp
int launch_seqw_bucket(int variant, uint32_t* slim, uint32_t* fat, const uint64_t* s_seeds, const uint64_t* f_seeds,
                       int d, int64_t w, int64_t z, const uint8_t* ops, KeySrc ks, int64_t n, int64_t* inc,
                       int64_t* result, cudaStream_t st) {
  int Z = 1;
  while (Z < z) Z <<= 1;
  if (d < 1 || (int64_t)d * Z > 32 || d > MAXD || w >= (int64_t(1) << 24)) return -1;
  SeqArgs a{};
  a.slim = slim;
  a.fat = fat;
  for (int i = 0; i < d; ++i) a.s_seeds.s[i] = s_seeds[i], a.f_seeds.s[i] = f_seeds[i];
  a.d = d;
  a.w = w;
  a.wp = 1;
  a.z = z;
  a.wm = make_mod((uint64_t)w);
  a.wpm = make_mod(1);
  a.zm = make_mod((uint64_t)z);
  a.ops = ops;
  a.keys = ks;
  a.n = n;
  a.inc = inc;
  a.result = result;
  note_launch();
  switch (Z) {
    case 1: seqw_bucket_k<1><<<1, 32, 0, st>>>(a, variant); break;
    case 2: seqw_bucket_k<2><<<1, 32, 0, st>>>(a, variant); break;
    case 4: seqw_bucket_k<4><<<1, 32, 0, st>>>(a, variant); break;
    case 8: seqw_bucket_k<8><<<1, 32, 0, st>>>(a, variant); break;
    case 16: seqw_bucket_k<16><<<1, 32, 0, st>>>(a, variant); break;
    default: seqw_bucket_k<32><<<1, 32, 0, st>>>(a, variant); break;
  }
  return check_launch("seqw_bucket");
}

int launch_seq_apply(int kind, int variant, uint32_t* slim, uint32_t* fat, uint32_t* dsub,
                     const uint64_t* s_seeds, const uint64_t* f_seeds, int d, int64_t w, int64_t wp, int64_t z,
                     const uint8_t* ops, KeySrc ks, const int64_t* true_counts, int64_t n, int64_t* inc,
                     int64_t* result, cudaStream_t st) {
  SeqArgs a;
  a.slim = slim;
  a.fat = fat;
  a.dsub = dsub;
  for (int i = 0; i < d; ++i) {
    a.s_seeds.s[i] = s_seeds ? s_seeds[i] : 0;
    a.f_seeds.s[i] = f_seeds ? f_seeds[i] : 0;
  }
  a.d = d;
  a.w = w;
  a.wp = wp > 0 ? wp : 1;
  a.z = z > 0 ? z : 1;
  a.wm = make_mod((uint64_t)w);
  a.wpm = make_mod((uint64_t)a.wp);
  a.zm = make_mod((uint64_t)a.z);
  a.ops = ops;
  a.keys = ks;
  a.true_counts = true_counts;
  a.exps = nullptr;
  a.gate = nullptr;
  a.rng_seed = 0;
  a.start_pos = 0;
  a.n = n;
  a.inc = inc;
  a.result = result;
  { note_launch(); seq_apply_k<<<1, 32, 0, st>>>(a, kind, variant); }
  return check_launch("seq_apply");
}

// Count (kind 5, counters = int32 table) and CML (kind 6, counters = u16 exponents)
int launch_seq_ext(int kind, void* counters, const uint64_t* seeds, int d, int64_t w, const uint8_t* ops, KeySrc ks,
                   int64_t n, const double* gate, uint64_t rng_seed, int64_t start_pos, int64_t* result,
                   cudaStream_t st) {
  SeqArgs a{};
  a.slim = kind == 5 ? static_cast<uint32_t*>(counters) : nullptr;
  a.exps = kind == 6 ? static_cast<uint16_t*>(counters) : nullptr;
  for (int i = 0; i < d; ++i) a.s_seeds.s[i] = seeds[i];
  a.d = d;
  a.w = w;
  a.wp = 1;
  a.z = 1;
  a.wm = make_mod((uint64_t)w);
  a.wpm = make_mod(1);
  a.zm = make_mod(1);
  a.ops = ops;
  a.keys = ks;
  a.gate = gate;
  a.rng_seed = rng_seed;
  a.start_pos = start_pos;
  a.n = n;
  a.result = result;
  { note_launch(); seq_apply_k<<<1, 32, 0, st>>>(a, kind, 0); }
  return check_launch("seq_apply");
}

}  // namespace sfk
