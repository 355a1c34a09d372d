/*
 * gmsketch_b200.h -- C ABI of the B200-native FastGM engine
 * (libgmsketch_b200.so, built for sm_100a).
 *
 * The reference (gmsketch 0.1.0, /root/reference/pkg/src/gmsketch) is pure
 * Python and has no FFI; its "operator API" is the Python function surface
 * of gmsketch/__init__.py:12-109.  Each entry point below names the
 * reference function(s) it replaces; the Python host package
 * paper_2302_05176_b200 binds them with ctypes and re-exports the
 * reference names.
 *
 * Conventions
 *  - Plain pointers and sizes only.  Pointers marked (device) must be CUDA
 *    device (or managed) memory; (host) pointers may be pageable or pinned.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *  - Element ids are unsigned 32- or 64-bit (id_bits = 32 | 64).  The
 *    reference keys its RNG on the id modulo 2**64 (randgen.py:115), so a
 *    negative Python id e is passed as e mod 2**64.
 *  - Weights are IEEE float or double (w_bits = 32 | 64); float weights are
 *    widened exactly to double, like float(np.float32(x)) in the reference.
 *  - Sketch registers: y (double, the value min_i E_ij / v_i) and s (uint64
 *    element id), k per sketch, row-major for batches.  An unset register
 *    has y = +inf and s = UINT64_MAX.
 *  - Return value: GM_OK (0) or one of the error codes below, which map 1:1
 *    onto the reference exception classes (errors.py:4-58); gm_last_error()
 *    returns a thread-local message for the last failing call.
 *  - Unless GM_FLAG_ASYNC is set, a call synchronises `stream` before it
 *    returns and reports data errors (bad weights, empty vectors).  With
 *    GM_FLAG_ASYNC the call only enqueues work; data errors are latched on
 *    the stream and returned by gm_stream_status().
 *  - Re-entrant per stream: scratch is kept per (device, stream); calls on
 *    different streams may run concurrently.
 */
#ifndef GMSKETCH_B200_H
#define GMSKETCH_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* error codes (reference exception in parentheses) */
#define GM_OK 0
#define GM_ERR_EMPTY_VECTOR 1       /* EmptyVectorError        sketch.py:172-174   */
#define GM_ERR_INVALID_WEIGHT 2     /* InvalidWeightError      sketch.py:54-64     */
#define GM_ERR_INVALID_PARAMETER 3  /* InvalidParameterError   sketch.py:151-157   */
#define GM_ERR_INCONSISTENT_WEIGHT 4 /* InconsistentWeightError stream.py:67-73    */
#define GM_ERR_INCOMPLETE 5         /* IncompleteSketchError   stream.py:132-134   */
#define GM_ERR_MISMATCHED 6         /* MismatchedSketchError   sketch.py:314-322   */
#define GM_ERR_CUDA 100             /* CUDA runtime failure (no reference class)   */
#define GM_ERR_NO_DEVICE 101        /* no sm_100 device visible                     */
#define GM_ERR_COMM 102             /* NCCL missing or a collective failed          */

/* flags */
#define GM_FLAG_ASYNC 0x1u       /* enqueue only; see gm_stream_status()           */
#define GM_FLAG_EXHAUSTIVE 0x2u  /* run every queue to k (sketch_naive semantics)  */
#define GM_FLAG_ACCUMULATE 0x4u  /* gm_sketch_elements: fold into y_io/s_io        */
/* 0x8u: reserved (was an experimental split schedule, removed) */
#define GM_FLAG_S32 0x10u        /* gm_sketch_csr_host: s_out is uint32 (32-bit ids) */
#define GM_FLAG_ONE_VECTOR 0x20u /* gm_sketch_csr_seeded: n_vec sketches of ONE vector */

/*
 * Multi-GPU register exchange (configs 4-5 sharded by element over N GPUs of
 * one node).  The reference's distributed form is "sketch
 * per site, merge centrally" (merge = estimate.py:103-125);
 * here every rank sketches its contiguous shard with gm_sketch_elements and
 * the k registers are combined in place over NCCL (NVLink / NVSwitch).
 * NCCL is opened at run time (libnccl.so.2); without it these return
 * GM_ERR_COMM and everything else still works.
 *   gm_comm_unique_id   rank 0 makes the id (gm_comm_id_bytes() bytes) and
 *                       shares it out of band (e.g. a torch.distributed
 *                       broadcast)
 *   gm_comm_init        one communicator per rank on the current device
 *   gm_allreduce_min_registers    two NCCL all-reduces with MIN (y; then
 *                       the ids of the ranks holding the minimum): the
 *                       register-wise (y, id) minimum -- smaller id wins a tie
 *                       of equal y (sketch.py:196-205)
 *   gm_allgather_merge_registers  NCCL all-gather of every rank's registers +
 *                       the device merge in rank order: merge([rank0, rank1,
 *                       ...]) exactly (earlier rank wins ties)
 * y (device, double[k]) and s (device, uint64[k]) are read and overwritten
 * with the merged sketch on every rank; enqueued on `stream`.
 */
int gm_comm_id_bytes(void);
int gm_comm_unique_id(void *id_out);
int gm_comm_init(const void *id, int nranks, int rank, void **comm_out);
int gm_comm_destroy(void *comm);
int gm_allreduce_min_registers(void *comm, double *y, uint64_t *s, int32_t k, void *stream);
int gm_allgather_merge_registers(void *comm, double *y, uint64_t *s, int32_t k, void *stream);

/* Library version (major*10000 + minor*100 + patch). */
int gm_version(void);
/* Debug builds (-DGM_DEBUG): first device bounds-check failure
 * ((line << 32) | code), else 0. */
int gm_debug_error(unsigned long long *out);
/* Thread-local message of the last failing call ("" if none). */
const char *gm_last_error(void);
/* Returns and clears the data error latched on `stream` by GM_FLAG_ASYNC
 * calls; synchronises the stream. */
int gm_stream_status(void *stream);

/* Lifecycle.  Scratch (device buffers, a page-locked readback word block)
 * is created lazily per (device, stream) by the first call on a stream and
 * reused by later calls on it.  gm_release_stream synchronises `stream` and
 * frees its scratch (call it before destroying a stream the library has
 * used); gm_finalize synchronises every device used and frees all scratch.
 * The library never retains caller memory.  gm_workspace_count: live
 * (device, stream) scratch sets.  (The reference is pure functions with no
 * retained state; this is the B200 engine's own housekeeping.) */
int gm_release_stream(void *stream);
int gm_finalize(void);
int gm_workspace_count(void);

/*
 * Batch of independent CSR vectors -> n_vec sketches.
 * Replaces sketch_fast / sketch_fast_counted (sketch.py:212-311) and, with
 * GM_FLAG_EXHAUSTIVE, sketch_naive / sketch_naive_counted (sketch.py:177-209),
 * applied to each vector; the reference has no batch call (its callers
 * loop, e.g. bench.py:264-292).
 *   ids, w      (device) n = offsets[n_vec] elements; ids distinct within a
 *               vector (WeightedVector keys, sketch.py:50-68)
 *   offsets     (device) n_vec+1 int64 CSR offsets
 *   y_out,s_out (device) n_vec*k
 *   emitted_out (device, nullable) n_vec arrivals computed per vector (the
 *               work counter of the *_counted variants; schedule-dependent)
 * Errors: GM_ERR_INVALID_PARAMETER (k outside [1, 65536], bad bits),
 *         GM_ERR_INVALID_WEIGHT, GM_ERR_EMPTY_VECTOR (a vector with no
 *         elements).
 */
int gm_sketch_csr(const void *ids, int id_bits, const void *w, int w_bits,
                  const int64_t *offsets, int64_t n_vec, int32_t k,
                  uint64_t global_seed, uint64_t stream_salt, uint32_t flags,
                  double *y_out, uint64_t *s_out, int64_t *emitted_out,
                  void *stream);

/* gm_sketch_csr with a global seed per vector (device array global_seeds[n_vec];
 * permutation seed = global_seeds[v] ^ stream_salt, as SeedScheme does,
 * randgen.py:72-95): one launch sketches the same vector under R seeds (R
 * independent sketches, e.g. for estimator variance) or a batch whose
 * vectors carry their own schemes.  With GM_FLAG_ONE_VECTOR, offsets holds
 * just [lo, hi] and all n_vec sketches are of that one vector (one per
 * seed; the vector is read once from HBM/L2, not replicated).  Needs k <=
 * the shared-memory register limit (k <= 4096 at 16 B per register, two
 * slots). */
int gm_sketch_csr_seeded(const void *ids, int id_bits, const void *w, int w_bits,
                         const int64_t *offsets, int64_t n_vec, int32_t k,
                         const uint64_t *global_seeds, uint64_t stream_salt,
                         uint32_t flags, double *y_out, uint64_t *s_out,
                         int64_t *emitted_out, void *stream);

/* Same contract with HOST buffers; copies in and out inside the call (page-
 * locked outputs are stored by the kernel directly).  With GM_FLAG_ASYNC the
 * call only enqueues: the caller keeps the buffers untouched until `stream`
 * is synchronised.  Alternating two streams pipelines batches: one batch's
 * input copy and first CTAs overlap the previous batch's tail.  With
 * GM_FLAG_S32 (32-bit ids only) s_out points to uint32 ids (an unset register
 * reads 0xFFFFFFFF): 12 instead of 16 bytes per register cross the bus.
 * A synchronous call with ONE vector of >= 4096 elements (GM_SINGLE_GRID_MIN)
 * runs on the grid-wide kernels of gm_sketch_elements (every SM) instead of
 * one CTA; same registers. */
int gm_sketch_csr_host(const void *ids, int id_bits, const void *w, int w_bits,
                       const int64_t *offsets, int64_t n_vec, int32_t k,
                       uint64_t global_seed, uint64_t stream_salt,
                       uint32_t flags, double *y_out, uint64_t *s_out,
                       int64_t *emitted_out, void *stream);

/*
 * One sketch over a large element set: a huge vector, or an (id, weight)
 * stream in which an id may repeat with the SAME weight (a repeat is a no-op
 * on the registers, stream.py:74-78).
 * Replaces sketch_stream / stream_update / stream_finalize
 * (stream.py:58-153) for bulk input and sketch_fast for vectors too large
 * for one CTA.
 *   ids, w      (device) n elements
 *   y_io, s_io  (device) k registers; read first when GM_FLAG_ACCUMULATE
 *   emitted_out (host, nullable) arrivals computed
 * Errors: GM_ERR_INVALID_PARAMETER, GM_ERR_INVALID_WEIGHT,
 *         GM_ERR_INCOMPLETE (n == 0 and no accumulated registers).
 * Always synchronises `stream` (the pass count is data-dependent).
 */
int gm_sketch_elements(const void *ids, int id_bits, const void *w, int w_bits,
                       int64_t n, int32_t k, uint64_t global_seed,
                       uint64_t stream_salt, uint32_t flags, double *y_io,
                       uint64_t *s_io, int64_t *emitted_out, void *stream);

/*
 * gm_sketch_elements without any host synchronisation, for a stream of
 * sketches: enqueues one pass that walks every element whose first arrival
 * is within the list bound tau_hi (R x the first threshold, K2),
 * so the sketch is complete unless the sampled weight was off by more than
 * that margin.  When the pass ends, the number of registers still unset is
 * written to *unset_out (DEVICE int); if it is non-zero after the stream is
 * synchronised, finish the sketch with gm_sketch_elements(...,
 * GM_FLAG_ACCUMULATE) over the same elements (registers already set stay
 * valid: an element's arrivals are folded idempotently).  Data errors are
 * latched and returned by gm_stream_status().  n >= 1; GM_FLAG_EXHAUSTIVE is
 * not accepted; GM_FLAG_ACCUMULATE is.
 */
int gm_sketch_elements_async(const void *ids, int id_bits, const void *w,
                             int w_bits, int64_t n, int32_t k,
                             uint64_t global_seed, uint64_t stream_salt,
                             uint32_t flags, double *y_io, uint64_t *s_io,
                             int32_t *unset_out, void *stream);

/* Same contract with HOST buffers. */
int gm_sketch_elements_host(const void *ids, int id_bits, const void *w,
                            int w_bits, int64_t n, int32_t k,
                            uint64_t global_seed, uint64_t stream_salt,
                            uint32_t flags, double *y_io, uint64_t *s_io,
                            int64_t *emitted_out, void *stream);

/*
 * Per-register minimum over n_sk sketches (row-major y_in/s_in, device),
 * strict '<' so the earlier sketch wins exact ties.  Replaces merge
 * (estimate.py:103-125); k/fingerprint compatibility (sketch.py:314-322) is
 * the caller's check.
 */
int gm_merge(const double *y_in, const uint64_t *s_in, int64_t n_sk,
             int32_t k, double *y_out, uint64_t *s_out, void *stream);

/*
 * Register-match counts of n_pairs sketch pairs (device, row-major
 * n_pairs*k): matches[p] = #{j : s_a[p,j] == s_b[p,j]}.  The numerator of
 * estimate_jaccard_p (estimate.py:47-55); the estimate is matches/k.
 */
int gm_match_count(const uint64_t *s_a, const uint64_t *s_b, int64_t n_pairs,
                   int32_t k, int32_t *matches, void *stream);

/* Cardinality estimates of n_sk sketches (estimate.py:90-100): sum_out[i] =
 * the correctly rounded sum of y[i*k .. i*k+k) (== math.fsum), card_out[i]
 * (nullable) = (k - 1) / sum_out[i].  Device arrays; asynchronous.  The
 * caller raises InvalidParameterError for k < 2 as the reference does. */
int gm_cardinality(const double *y, int64_t n_sk, int32_t k, double *sum_out,
                   double *card_out, void *stream);

/* K0 test surface (device arrays of length n): uniform_open
 * (randgen.py:107-119) and the permutation draw j in [z, k]
 * (rand_int_between(scheme, e, z, z, k), randgen.py:122-143). */
int gm_uniform_open_batch(const uint64_t *global_seeds, const uint64_t *elements,
                          const uint64_t *steps, int64_t n, double *out,
                          void *stream);
int gm_perm_draw_batch(const uint64_t *perm_seeds, const uint64_t *elements,
                       const uint64_t *steps, const uint32_t *ks, int64_t n,
                       uint32_t *out, void *stream);
/* rand_int_between(scheme, e, step, lo, hi) over ANY range (randgen.py:122-143):
 * out[i] = (result - lo), the offset in [0, m), m = m_minus_1[i] + 1 <= 2^64
 * (m_minus_1 = UINT64_MAX means m = 2^64); keys (perm_seeds[i], elements[i]
 * mod 2^64, steps[i] mod 2^64).  (device) arrays; synchronises. */
int gm_rand_int_between_batch(const uint64_t *perm_seeds, const uint64_t *elements,
                              const uint64_t *steps, const uint64_t *m_minus_1,
                              int64_t n, uint64_t *out, void *stream);

/* ElementQueueState / next_order_statistic (randgen.py:210-271) on the device:
 * n queues of k customers each advance `steps` emissions.  Queue i is element
 * elements[i] with weight weights[i], z0[i] order statistics already emitted,
 * the last at time b0[i]; perm + i*k is its Fisher-Yates array (values 1..k,
 * swapped in place).  Emission q of queue i: t_out[i*steps+q] (arrival time)
 * and s_out[i*steps+q] (server, 1..k); b_out[i] = the last time.  The caller
 * keeps z0[i] + steps <= k.  (device) arrays; asynchronous. */
int gm_queue_advance_batch(const uint64_t *elements, const double *weights, const int32_t *z0,
                           const double *b0, int64_t n, int32_t k, int32_t steps,
                           uint64_t global_seed, uint64_t stream_salt, uint32_t *perm,
                           double *t_out, uint32_t *s_out, double *b_out, void *stream);

/* Arithmetic self-checks (device).
 * gm_arith_check: over n keyed random inputs, counts[0] = #(branch-free
 * divide != IEEE __ddiv_rn) on the fast weight range, counts[1] = #(device
 * log_pos more than 1 ulp from CUDA's log).  counts: 2 device u64.
 * gm_log_batch: out[i] = device natural log of x[i] > 0 (device arrays); the
 * log every walker uses in -log(u) (randgen.py:186, math.log in the
 * reference).  Both synchronise `stream`. */
int gm_arith_check(int64_t n, uint64_t seed, unsigned long long *counts,
                   void *stream);
int gm_log_batch(const double *x, int64_t n, double *out, void *stream);

/* Stream checks for bulk (id, weight) pairs (device arrays; stream.py:58-78
 * for every item at once): *first_bad = index of the first item whose weight
 * is not finite, > 0 and >= 1e-300 (InvalidWeightError), *first_conflict =
 * index of the first item whose id appeared earlier with another weight
 * (InconsistentWeightError); -1 when there is none.  With uniq_ids/uniq_w
 * (device arrays of capacity n, same types as the input; both or neither)
 * the first occurrence of every id is compacted there (any order) and
 * *n_uniq is its count: the skip_duplicates input of gm_sketch_elements.
 * Synchronises `stream`. */
int gm_check_pairs(const void *ids, int id_bits, const void *w, int w_bits,
                   int64_t n, int64_t *first_bad, int64_t *first_conflict,
                   void *uniq_ids, void *uniq_w, int64_t *n_uniq,
                   void *stream);

/* Exact-y finalize (host memory only; no CUDA): y_io[v*k + j] := the
 * arrival time the reference computes for register j of CSR vector v,
 * given its winning element s[v*k + j] (from gm_sketch_csr* /
 * gm_sketch_elements), by walking that element's queue with glibc log and
 * IEEE double arithmetic in the reference's operation order
 * (randgen.py:158-207).  A host cross-check: the device's y already carries
 * these bits (its log is glibc's, gm_glibc_log.cuh), and no entry point calls
 * it.  Every
 * s must name an element of its vector (else GM_ERR_MISMATCHED).  For a
 * stream, pass n_vec = 1 and offsets {0, n}.  n_threads <= 0: all host
 * threads.  Replaces the float equality of GumbelMaxSketch
 * (sketch.py:118-136) for sketches built on the device. */
int gm_exact_y(const void *ids, int id_bits, const void *w, int w_bits,
               const int64_t *offsets, int64_t n_vec, int32_t k,
               uint64_t global_seed, uint64_t stream_salt, const uint64_t *s,
               double *y_io, int32_t n_threads);

/* Work counters of a library built with -DGM_STATS (tools/stats.py): copies
 * and clears 16 u64 host words; GM_ERR_INVALID_PARAMETER in normal builds. */
int gm_stats_read(unsigned long long *out16);
/* Slot events of a -DGM_EVENTS build (tools/timeline.py): ev_out up to
 * 32768 x 2 u64 (globaltimer ns, vector | pass << 32 | kind << 40 | cta << 48
 * | slot << 60; kind 0 load, 1 written, 2 re-opened), *n_out their count;
 * clears them.  GM_ERR_INVALID_PARAMETER in normal builds. */
int gm_trace_read(unsigned long long *ev_out, unsigned *n_out);

/* Diagnostics.
 * gm_probe_arrival_rate: n_threads threads each walk C element queues for
 * `iters` exact arrivals apiece (iters | C << 24, C = 1, 2 or 4; C = 0 means
 * 2), with the lane step's own arithmetic (uniform hash, glibc-clone log from
 * a shared-memory table, rounded product, branch-free divide, prefix add,
 * permutation hash + 64-bit Barrett reduction) and no pruning, tables or
 * registers; the measured rate is the compute roofline of the sketch kernels
 * (DESIGN.md).  sink: 1 device double.  Asynchronous.
 * gm_count_arrivals_csr: counts[v] = number of arrivals t <= tau[v] over the
 * elements of CSR vector v (device arrays); the algorithmic survivor count.
 * Synchronises `stream`. */
int gm_probe_arrival_rate(int64_t n_threads, int32_t iters, int32_t k,
                          double *sink, void *stream);
int gm_count_arrivals_csr(const void *ids, int id_bits, const void *w,
                          int w_bits, const int64_t *offsets, int64_t n_vec,
                          int32_t k, uint64_t global_seed, const double *tau,
                          unsigned long long *counts, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* GMSKETCH_B200_H */
