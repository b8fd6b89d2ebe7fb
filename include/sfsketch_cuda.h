/*
 * sfsketch_cuda.h — C ABI of the B200-native SF sketch hot path.
 *
 * Every entry point replaces one numba kernel of the reference package
 * (/root/reference/pkg/src/sfsketch/_kernels.py); the comment on each
 * declaration cites the reference interface (file:line) it stands in for.
 *
 * Conventions (mirroring _kernels.py:1-16 and SURVEY.md §8(b)):
 *   - Seeds (slim_seeds, fat_seeds, seeds) are HOST arrays of d uint64 values
 *     (hashing.seed_array, hashing.py:132-137); they travel to the kernels by
 *     value. Every other array argument is a DEVICE pointer owned by the
 *     caller; state
 *     arrays (counters, slim, fat, inc_counts) are mutated in place.
 *   - Counters are uint32, row-major (d, w); the bucketed fat is (d, w, z)
 *     C-order; tallies (inc_counts) are int64[d]; query estimates int64.
 *   - Keys are described by (keys, key_kind, rec_len):
 *       SFK_KEY_U64     uint64[n] (the reference's native key dtype)
 *       SFK_KEY_U32     uint32[n], zero-extended to u64 (_ops.py:21)
 *       SFK_KEY_RECORD  uint8[n * rec_len] packed byte records, hashed to a
 *                       u64 key with FNV-1a-64 + finalize64, identical to
 *                       hashing.key_from_string (hashing.py:124-129) for
 *                       ASCII/UTF-8 bytes.
 *   - ops are uint8[n], 0 = insert, 1 = delete (_kernels.py:28-29).
 *   - Apply entry points never fail on sketch semantics: they write
 *     {status, op_index, n_ins} into the device array `result` (int64[3])
 *     with status codes OK=0 PHANTOM=1 SATURATED=2 UNSUPPORTED=3
 *     (_kernels.py:21-24). A batch aborts at its first failing op: ops
 *     before it are applied, the failing op leaves no trace.
 *   - The int return value is a CUDA error code (0 = success), distinct
 *     from the sketch status; sfk_last_error() describes it.
 *   - Everything is stream-ordered on `stream` (a cudaStream_t passed as
 *     void*). Apply calls need exclusive access to their state; queries on a
 *     quiesced sketch may run concurrently on other streams or GPUs.
 *   - Scratch memory is caller-provided: query sfk_*_workspace_size() and
 *     pass a device buffer of at least that many bytes.
 */
#ifndef SFSKETCH_CUDA_H
#define SFSKETCH_CUDA_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SFK_KEY_U64 0
#define SFK_KEY_U32 1
#define SFK_KEY_RECORD 2

#define SFK_OK 0
#define SFK_PHANTOM 1
#define SFK_SATURATED 2
#define SFK_UNSUPPORTED 3
/* an op code other than 0 (insert) / 1 (delete): nothing of the batch is
 * applied and op_index is the first such op (the reference rejects the batch
 * in normalize_stream before any kernel runs, _ops.py:27-34, with
 * ConfigurationError). Checked on the device by sfk_sf_apply, sfk_cm_apply
 * and sfk_cu_apply. */
#define SFK_BAD_OPCODE 4

/* SF variant codes: sf.py:57 (_FLAT_VARIANT_CODE) and sf.py:171-172 (mode) */
#define SFK_VARIANT_SF1 1
#define SFK_VARIANT_SF2 2
#define SFK_VARIANT_SF3 3
#define SFK_VARIANT_SF4 4
#define SFK_VARIANT_SFF 6

/* apply flags: SFK_FLAG_SEQUENTIAL forces the exact one-thread device engine
 * (the reference loop replayed in order) instead of the parallel engine; the
 * parity tests use it to cross-check the two on the GPU. */
#define SFK_FLAG_SEQUENTIAL 1

/* Threading: the compute entry points keep no state between calls (all
 * scratch is the caller's workspace) and may run concurrently on different
 * streams and host threads; sfk_last_error() is per host thread. The
 * diagnostics below (engine timing / trace / stats, sfk_query_path) are
 * process-global switches for benchmarks and tests, not for concurrent use. */
int sfk_abi_version(void);
const char* sfk_last_error(void);

/* cudaStreamSynchronize(stream): the Python layer's wait before it reads a
 * result triple from pinned host memory (no torch stream object needed). */
int sfk_stream_sync(void* stream);

/* Batches of 1..ops ops (default 32) go to the exact one-thread device engine
 * (one launch, no host read-back) instead of the parallel pipeline, whose
 * fixed cost dominates tiny batches: SF, CM, CU, Count, CML and oracle-
 * assisted applies. 0 turns it off;
 * a negative value only reads. Returns the previous value. Process-global. */
int64_t sfk_small_batch_ops(int64_t ops);

/* Diagnostics: number of kernels this library has launched in the process
 * (its own kernels; CUB's internal radix-sort/scan launches excluded). */
unsigned long long sfk_launch_count(void);

/* Diagnostics of the ordered slim engine, summed over launches since the last
 * reset: out8 = {words on the gap path, words on the steady path, words
 * replayed op by op, replay cycles, runs executed, warp iterations, long-run
 * pieces applied, ops finished by long-run pieces}. */
int sfk_engine_stats(unsigned long long* out8, int reset);

/* Bench instrumentation: when on, CUDA events bracket every launch of the
 * ordered slim engine kernel; sfk_engine_last_ms() synchronises on the last
 * one and returns its duration in ms (-1 if none was recorded). */
int sfk_engine_timing(int on);

/* Diagnostics: with SFK_ENGINE_TRACE set in the environment the engine
 * records {claim, ready, done} globaltimer stamps (ns) per run; this copies
 * the last launch's stamps for the first `runs` runs to host memory. */
int sfk_engine_trace(unsigned long long* host_out, size_t runs);
float sfk_engine_last_ms(void);

/* Workload utility (no reference counterpart; SURVEY.md §8(d) cfg 5): keys
 * t0 .. t0+n-1 of the counter-based query stream of
 * paper_1701_04148_b200.workloads.query_keys, generated on the device.
 * present: uint32[v] keys in draw order; sorted_present: the same sorted;
 * cdf: float64[v] Zipf CDF or NULL for uniform ranks. */
int sfk_gen_query_keys(uint64_t seed, const uint32_t* present, const uint32_t* sorted_present, uint32_t v,
                       const double* cdf, int64_t t0, int64_t n, uint32_t* out, void* stream);

/* Replaces _kernels.mix_batch (_kernels.py:56-59): out[t] = finalize64(keys[t]). */
int sfk_mix_batch(const uint64_t* keys, int64_t n, uint64_t* out, void* stream);

/* Key materialisation for any key kind (hashing.py:124-129 for records). */
int sfk_load_keys(const void* keys, int key_kind, int rec_len, int64_t n, uint64_t* out, void* stream);

/* Replaces _kernels.min_query (_kernels.py:229-241), called from
 * SfSketch.query_many (sf.py:189-193), CmSketch/CuSketch.query_many
 * (baselines.py:83-87, 167-171) and CollectorSketch.query_many
 * (serialize.py:140-145). out[t] = min_i counters[i, h_i(key_t)]. */
int sfk_min_query(const uint32_t* counters, const uint64_t* seeds, int d, int64_t w,
                  const void* keys, int key_kind, int rec_len, int64_t n, int64_t* out,
                  void* stream);

/* Host-buffer form of sfk_min_query: the reference's query_many takes and
 * returns host arrays (sf.py:189-193, _kernels.py:229-241; its ctypes binding
 * is INTEGRATION.md's query_many). keys_host and out_host are host pointers
 * (pinned or pageable); counters and seeds as in sfk_min_query. Blocks until
 * out_host holds every estimate. Work on `stream` issued before the call is
 * complete before the slim is read. The batch flows through H2D -> query
 * kernel -> D2H in chunks; the estimates cross PCIe narrowed (u16 codes when
 * the slim has at most 2048 distinct counter values >= 0xF800, else u32) and
 * host threads widen them into out_host. Bit-identical to sfk_min_query. */
int sfk_min_query_host(const uint32_t* counters, const uint64_t* seeds, int d, int64_t w,
                       const void* keys_host, int key_kind, int rec_len, int64_t n, int64_t* out_host,
                       void* stream);

/* sfk_min_query_host for a batch whose first n_dev keys the caller has
 * already copied to the device (keys_dev, the same bytes as keys_host's
 * prefix, the copy ordered before `stream`'s work): chunks wholly inside the
 * prefix are queried in place without an H2D, so the caller can upload them
 * while the sketch is still being built (SfSketch.stage_query_keys). No
 * reference counterpart (the reference's query_many, sf.py:189-193, takes one
 * host array); keys_host must still hold all n keys. n_dev = 0 is
 * sfk_min_query_host. */
int sfk_min_query_host_staged(const uint32_t* counters, const uint64_t* seeds, int d, int64_t w,
                              const void* keys_host, int key_kind, int rec_len, int64_t n, int64_t* out_host,
                              const void* keys_dev, int64_t n_dev, void* stream);

/* Tuning of sfk_min_query_host (no reference counterpart). what:
 *   0 = keys per chunk (default 2^22);
 *   1 = wire (0 auto, 1 int64, 2 u32, 3 u16 codes where exact, else u32);
 *   2 = every value-th chunk returns int64 directly when out_host is pinned
 *       (0 = never, default);
 *   3 = host threads (0 = 3/4 of the hardware threads / LOCAL_WORLD_SIZE);
 *   4 = chunks in flight (2-16, default 8);
 *   5 = the wire the last call used (read only).
 * value < 0 only reads. Returns the previous value, or -1 for an unknown key
 * or value. */
int64_t sfk_host_query_config(int what, int64_t value);

/* Query kernel selection (no reference counterpart: the reference has one
 * numba loop). mode: 0 = automatic (default), 1 = L2 gathers, 2 = whole table
 * in one SM's shared memory (only if it fits), 3 = row-partitioned cluster
 * (d CTAs, one row each, DSMEM min-reduction; only for 2 <= d <= 8 and a row
 * that fits), 4 = its warp-pipelined form (u32 or u64 keys, d in {2, 4, 8},
 * 16-B aligned keys and output, >= one warp-tile of keys; otherwise as 3); a
 * mode that does not apply falls back to the L2 path. A
 * negative mode only reads. Returns the previous mode. sfk_query_last_path()
 * returns the path (1-4) the last sfk_min_query launch took. */
int sfk_query_path(int mode);

/* Small-batch engine selection (no reference counterpart). SFF / SF4 batches
 * of at most `ops` ops (default 24; 0 = off) run on the warp-cooperative
 * exact engine: ops in stream order, each op's d x z counter reads in one
 * round of parallel loads, one launch and no host round trip. A negative
 * value only reads. Returns the previous value. */
int64_t sfk_warp_batch_ops(int64_t ops);

/* Medium-batch engine selection (no reference counterpart). SFF / SF4 batches
 * above sfk_warp_batch_ops() and up to `ops` ops (default 2048; at most 8192
 * (op, row) pairs, z <= 8) run on the block engine: one 1024-thread CTA sorts,
 * walks the fat and replays the slim updates as a dataflow in shared memory,
 * in one launch and with no workspace. A negative value only reads. Returns
 * the previous value. */
int64_t sfk_block_batch_ops(int64_t ops);

/* Diagnostics: globaltimer stamps (ns) at the block engine's phase boundaries
 * in its last launch (start, sorted, scanned, fat pass, replayed, done). */
int sfk_blk_profile(unsigned long long* out6);
int sfk_query_last_path(void);

/* Two-phase form of sfk_min_query (no reference counterpart; same
 * estimates). sfk_query_index writes each key's bucket index for every row
 * as uint16 (w <= 65536): idx[r * n + t] = h_r(key_t). It reads no counters,
 * so it may run while the sketch is still being updated on another stream.
 * sfk_min_query_idx then computes out[t] = min_r counters[r, idx[r * n + t]]. */
int sfk_query_index(const uint64_t* seeds, int d, int64_t w, const void* keys, int key_kind, int rec_len, int64_t n,
                    uint16_t* idx, void* stream);
int sfk_min_query_idx(const uint32_t* counters, int d, int64_t w, const uint16_t* idx, int64_t n, int64_t* out,
                      void* stream);

/* Replaces _kernels.cm_apply (_kernels.py:62-88), called from
 * CmSketch.apply_ops (baselines.py:72-78). */
size_t sfk_cm_workspace_size(int d, int64_t w, int64_t n);
int sfk_cm_apply(uint32_t* counters, const uint64_t* seeds, int d, int64_t w, const uint8_t* ops,
                 const void* keys, int key_kind, int rec_len, int64_t n, int64_t* inc_counts,
                 int64_t* result, void* workspace, size_t workspace_bytes, int flags, void* stream);

/* Raw signed count-min update (no reference counterpart; the building block
 * of stream-sharded CM builds, distributed.sharded_cm_apply, which replaces
 * one _kernels.cm_apply call, _kernels.py:62-88, by per-rank shards):
 * counters[i, h_i(key_t)] += 1 for an insert and -= 1 for a delete, modulo
 * 2^32, with no saturation or phantom checks and no tallies. The caller
 * proves that no op of the whole batch can fail (sfk_cm_apply's precheck:
 * max counter + inserts <= 2^32 - 1, and no deletes or min counter >=
 * deletes), so summing the shards' deltas equals the sequential apply.
 * d <= 8. Warp-aggregated atomics; asynchronous on `stream`. */
int sfk_cm_delta(uint32_t* counters, const uint64_t* seeds, int d, int64_t w, const uint8_t* ops,
                 const void* keys, int key_kind, int rec_len, int64_t n, void* stream);

/* Replaces _kernels.cu_apply (_kernels.py:91-115), called from
 * CuSketch.apply_ops (baselines.py:156-162). */
size_t sfk_cu_workspace_size(int d, int64_t w, int64_t n);
int sfk_cu_apply(uint32_t* counters, const uint64_t* seeds, int d, int64_t w, const uint8_t* ops,
                 const void* keys, int key_kind, int rec_len, int64_t n, int64_t* inc_counts,
                 int64_t* result, void* workspace, size_t workspace_bytes, int flags, void* stream);

/* Replaces _kernels.sf_flat_apply (_kernels.py:244-315; variants 1, 2, 3)
 * and _kernels.sf_bucket_apply (_kernels.py:318-384; SF4 = mode 0,
 * SFF = mode 1), called from SfSketch.apply_ops (sf.py:149-184).
 *   variant  SFK_VARIANT_*; fat is (d, w_prime) for SF1/SF2/SF3 and
 *            (d, w, z) for SF4/SFF; dsub is the (d, w) deletion sub-sketch
 *            for SF2, else NULL.
 *   slim_seeds = seed_array(master, 0, d); fat_seeds = seed_array(master, d, d)
 *   (sf.py:115-116), except SF3 whose fat uses the slim seeds (sf.py:130). */
size_t sfk_sf_workspace_size(int variant, int d, int64_t w, int64_t w_prime, int z, int64_t n);
int sfk_sf_apply(int variant, uint32_t* slim, uint32_t* fat, uint32_t* dsub,
                 const uint64_t* slim_seeds, const uint64_t* fat_seeds, int d, int64_t w,
                 int64_t w_prime, int z, const uint8_t* ops, const void* keys, int key_kind,
                 int rec_len, int64_t n, int64_t* inc_counts, int64_t* result, void* workspace,
                 size_t workspace_bytes, int flags, void* stream);

/* Replaces _kernels.oracle_slim_apply (_kernels.py:387-411), called from
 * SfSketch.oracle_assisted_apply (sf.py:199-229). true_counts: int64[n] on
 * the device. The ordered engine replays the batch (gate: m <
 * np.uint64(true count)); a batch holding a count that is negative or above
 * 2^32 - 1 while a slim cell could reach 2^32 - 1 (checked on the device)
 * runs in the exact sequential engine. */
size_t sfk_oracle_workspace_size(int d, int64_t w, int64_t n);
int sfk_oracle_slim_apply(uint32_t* slim, const uint64_t* seeds, int d, int64_t w, const void* keys,
                          int key_kind, int rec_len, const int64_t* true_counts, int64_t n,
                          int64_t* inc_counts, int64_t* result, void* workspace, size_t workspace_bytes,
                          int flags, void* stream);

/* Replaces _kernels.count_apply (_kernels.py:118-146), called from
 * CountSketch.apply_ops (baselines.py:115-119). counters: int32 (d, w).
 * result = {status, op_index, n_ins} (no tallies: the reference keeps none).
 * Batches that cannot reach +-2^31 (checked on the device) are one pass of
 * warp-aggregated atomics; the others run in the exact sequential engine. */
size_t sfk_count_workspace_size(int d, int64_t w, int64_t n);
int sfk_count_apply(int32_t* counters, const uint64_t* seeds, int d, int64_t w, const uint8_t* ops,
                    const void* keys, int key_kind, int rec_len, int64_t n, int64_t* result,
                    void* workspace, size_t workspace_bytes, int flags, void* stream);
/* Replaces _kernels.count_query (_kernels.py:149-179): median of the d
 * sign-corrected reads (even d: mean of the central pair, half away from
 * zero), clamped at 0, as int64. */
int sfk_count_query(const int32_t* counters, const uint64_t* seeds, int d, int64_t w, const void* keys,
                    int key_kind, int rec_len, int64_t n, int64_t* out, void* stream);

/* Replaces _kernels.cml_apply (_kernels.py:182-211), called from
 * CmlSketch.apply_ops (baselines.py:219-231). exps: uint16 (d, w).
 * gate: device float64[65536], gate[c] = base ** -c as the host's libm pow
 * computes it (numba's float ** lowers to the same call). start_pos = the
 * sketch's insertions_seen before the batch (the coin-flip stream index).
 * Runs in the ordered engine when the gate is non-increasing and the 0xFFFF
 * exponent cannot be raised within the batch (gate[65535] == 0, or the
 * largest exponent + n < 0xFFFF; checked on the device), else in the exact
 * sequential engine. */
size_t sfk_cml_workspace_size(int d, int64_t w, int64_t n);
int sfk_cml_apply(uint16_t* exps, const uint64_t* seeds, int d, int64_t w, const uint8_t* ops,
                  const void* keys, int key_kind, int rec_len, int64_t n, const double* gate,
                  uint64_t rng_seed, int64_t start_pos, int64_t* result, void* workspace,
                  size_t workspace_bytes, int flags, void* stream);
/* Replaces _kernels.cml_min_exp (_kernels.py:214-226) and, when value_table
 * (device int64[65536], the reference's cml_value of every exponent) is
 * given, the decode of CmlSketch.query_many (baselines.py:236-238). */
int sfk_cml_query(const uint16_t* exps, const uint64_t* seeds, int d, int64_t w, const void* keys,
                  int key_kind, int rec_len, int64_t n, const int64_t* value_table, int64_t* out,
                  void* stream);

/* Synthetic streams (workloads.generate, workloads.py:92-131) on the device.
 * sfk_pcg64_draws: draws [offset, offset + n) of numpy's Generator(PCG64)
 * stream given its seeded 128-bit state / increment (host: bit_generator
 * .state), as random() doubles, or, with a device CDF of v entries, as
 * Zipf ranks searchsorted(cdf, u, side="right"). sfk_interleave_deletions:
 * _kernels.interleave_deletions (_kernels.py:427-467), one device thread
 * (the walk is sequential). Keys are then sfk_mix_batch(ranks). */
int sfk_pcg64_draws(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t offset,
                    int64_t n, const double* cdf, int64_t v, int64_t* ranks, double* uniforms,
                    void* stream);
/* numpy's Generator.integers(0, v, dtype=int64) for 1 <= v <= 2^32 from the
 * same stream: n samples starting at 64-bit draw offset64 (Lemire's method
 * with rejection over the low-then-high 32-bit halves of each draw; accepted
 * positions compacted in parallel). *next_offset64 (host) = the stream
 * position after them (numpy drops a half-used 64-bit draw). */
size_t sfk_pcg64_bounded_workspace_size(int64_t n, int64_t v);
int sfk_pcg64_bounded(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t offset64,
                      int64_t n, int64_t v, int64_t* out, int64_t* next_offset64, void* workspace,
                      size_t workspace_bytes, void* stream);
size_t sfk_interleave_workspace_size(int64_t v);
int sfk_interleave_deletions(const int64_t* candidates, const double* decide, const double* pick,
                             double p, int64_t n, int64_t v, uint8_t* ops, int64_t* ranks,
                             void* workspace, size_t workspace_bytes, void* stream);

/* Trace ingestion (workloads.read_trace / load_trace, workloads.py:132-172):
 * "OP,key" text lines parsed on the device. Phase 1 fills per-line arrays
 * (device, nbytes + 1 entries each): line_pos (byte offset), status (0 blank
 * or comment, 1 op, 2 "expected 'OP,key'", 3 unknown op token, 4 bad key,
 * 5 key out of 64-bit range, 6 non-ASCII line left to the host), op, key;
 * info (host int64[3]) = {lines, first error line (0-based) or -1, non-ASCII
 * lines}. Phase 2 compacts the status-1 lines into ops / keys (device) and
 * returns their count in *n_out (host). Universal newlines, str.strip()
 * whitespace, int(key, 10) syntax (sign, digit-group underscores). */
size_t sfk_trace_workspace_size(int64_t nbytes);
int sfk_trace_parse_lines(const uint8_t* text, int64_t nbytes, int64_t* line_pos, uint8_t* status,
                          uint8_t* op, uint64_t* key, int64_t* info, void* workspace,
                          size_t workspace_bytes, void* stream);
int sfk_trace_compact(const uint8_t* status, const uint8_t* op, const uint64_t* key, int64_t nlines,
                      uint8_t* ops, uint64_t* keys, int64_t* n_out, void* workspace,
                      size_t workspace_bytes, int64_t nbytes, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SFSKETCH_CUDA_H */
