/*
 * gm_oracle.h -- CPU restatement of the reference FastGM path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the CUDA
 * library, the Python host package) may include, link or call this code.
 * It is used by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg, and only as the checker.
 *
 * Every function restates a reference function (paths relative to
 * /root/reference/pkg/src/gmsketch); arithmetic follows the reference
 * operation for operation, and log() is glibc libm's log, the same
 * function CPython's math.log calls, so the restatement is bit-exact
 * with the Python reference (pinned by tests/test_oracle_golden.py).
 */
#ifndef GM_ORACLE_H
#define GM_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  GMO_OK = 0,
  GMO_EMPTY_VECTOR = 1,        /* EmptyVectorError        sketch.py:172-174 */
  GMO_INVALID_WEIGHT = 2,      /* InvalidWeightError      sketch.py:57-64   */
  GMO_INVALID_PARAMETER = 3,   /* InvalidParameterError   sketch.py:151-157 */
  GMO_INCONSISTENT_WEIGHT = 4, /* InconsistentWeightError stream.py:67-73   */
  GMO_INCOMPLETE = 5,          /* IncompleteSketchError   stream.py:132-134 */
  GMO_NO_MEMORY = 6
};

/* randgen.py:64-69 */
uint64_t gmo_mix64(uint64_t x);
/* randgen.py:94-95 */
uint64_t gmo_fingerprint(uint64_t global_seed, uint64_t stream_salt);
/* randgen.py:98-104 */
uint64_t gmo_derive_seed(uint64_t master, uint64_t index);
/* randgen.py:107-119 (step >= 1) */
double gmo_uniform_open(uint64_t global_seed, uint64_t element, uint64_t step);
/* randgen.py:122-143 (step >= 1, lo <= hi, hi - lo < 2^64 - 1) */
uint64_t gmo_rand_int_between(uint64_t perm_seed, uint64_t element,
                              uint64_t step, uint64_t lo, uint64_t hi);
/* randgen.py:158-207 over the whole queue (z0=0, z1=k): k times and
 * 1-based servers, in emission order. */
void gmo_run_queue_full(uint64_t global_seed, uint64_t perm_seed,
                        uint64_t element, double weight, int32_t k,
                        double *times, int32_t *servers);
/* CPython math.fsum (exactly rounded sum), used at sketch.py:69 and
 * estimate.py:100. */
double gmo_fsum(const double *x, int64_t n);

/* sketch.py:183-209.  Elements are processed in the given order (the
 * reference iterates WeightedVector.items(), i.e. ascending id; callers
 * sort). */
int gmo_sketch_naive(const uint64_t *ids, const double *w, int64_t n,
                     int32_t k, uint64_t global_seed, uint64_t stream_salt,
                     double *y, uint64_t *s, int64_t *emitted);
/* sketch.py:218-311 (FastSearch + FastPrune), same emitted count as the
 * reference when the input is sorted by id. delta<=0 means delta=k. */
int gmo_sketch_fast(const uint64_t *ids, const double *w, int64_t n,
                    int32_t k, int64_t delta, uint64_t global_seed,
                    uint64_t stream_salt, double *y, uint64_t *s,
                    int64_t *emitted);
/* stream.py:30-153 (sketch_stream).  On InconsistentWeightError the index
 * of the offending item is stored in *err_index. */
int gmo_sketch_stream(const uint64_t *ids, const double *w, int64_t n,
                      int32_t k, uint64_t global_seed, uint64_t stream_salt,
                      int skip_duplicates, double *y, uint64_t *s,
                      int64_t *emitted, int64_t *err_index);
/* A batch of CSR vectors sketched independently on `threads` host
 * threads.  mode 0: sketch_fast on each vector sorted by id (requires
 * distinct ids); mode 1: sketch_stream over each vector in given order.
 * y/s are n_vec*k row-major.  emitted (nullable) is per vector. */
int gmo_sketch_csr(const uint64_t *ids, const double *w,
                   const int64_t *offsets, int64_t n_vec, int32_t k,
                   uint64_t global_seed, uint64_t stream_salt, int mode,
                   int threads, double *y, uint64_t *s, int64_t *emitted);
/* estimate.py:103-125: per register strict '<', earlier sketch wins ties.
 * y_in/s_in are n_sk*k row-major. */
/* uniform_open(seed, i0 + i, 1) and glibc log of it, i < n */
void gmo_log_uniforms(uint64_t seed, int64_t i0, int64_t n, double *u_out, double *log_out);
void gmo_merge(const double *y_in, const uint64_t *s_in, int64_t n_sk,
               int32_t k, double *y_out, uint64_t *s_out);

#ifdef __cplusplus
}
#endif
#endif
