// gm_capi.cu -- the C ABI (include/gmsketch_b200.h) over the sm_100a kernels.
//
// Host orchestration only: argument checks, per-(device, stream) scratch,
// launch configuration, the pass loop of gm_sketch_elements, error mapping.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <limits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <utility>

#include "../../include/gmsketch_b200.h"
#include "gm_csr.cuh"
#include "gm_csr4.cuh"
#include "gm_pairs.cuh"
#include "gm_comm.cuh"

#include <cub/device/device_scan.cuh>

using namespace gmk;

// registers per sketch: up to 2^24 (256 MB of (y, s) registers; queues of more
// than 65536 customers run on the grid-wide kernels with 64-bit Fisher-Yates words)
constexpr int32_t GM_K_MAX = 1 << 24;

namespace {

thread_local char g_msg[512] = "";

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_msg, sizeof(g_msg), fmt, ap);
  va_end(ap);
  return code;
}

#define CK(call)                                                                      \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess) {                                                          \
      (void)cudaGetLastError(); /* do not leave a non-sticky error for other libs */  \
      return fail(GM_ERR_CUDA, "%s failed: %s", #call, cudaGetErrorString(e_));       \
    }                                                                                 \
  } while (0)

struct Workspace {
  int* counters = nullptr;                 // [0] vector ticket, [1] unset registers
  unsigned long long* err = nullptr;       // latched data error
  unsigned long long* ull = nullptr;       // [0] heavy count, [1] emitted total
  double* dbl = nullptr;                   // [0] tau, [1] sampled weight, [2] sampled distinct weight, [3] tau_hi
  unsigned long long* host = nullptr;      // pinned readback / upload (16 words)
  Reg* regs = nullptr;
  size_t regs_cap = 0;
  u64* heavy = nullptr;
  size_t heavy_cap = 0;
  u32* dense = nullptr;
  size_t dense_cap = 0;
  u32* csr_dense = nullptr;                // CSR warp-walker dense arrays (stamped)
  size_t csr_dense_cap = 0;
  Surv* surv = nullptr;                    // K2 filter survivors (id, weight)
  size_t surv_cap = 0;
  unsigned long long* sample_set = nullptr;  // K2 weight-sample id set
  size_t sample_set_cap = 0;
  double* sample_part = nullptr;           // K2 weight-sample per-block partial sums
  size_t sample_part_cap = 0;
  void* stage = nullptr;                   // device staging for *_host calls
  size_t stage_cap = 0;
  u64* pt_keys = nullptr;                  // gm_check_pairs id table
  size_t pt_keys_cap = 0;
  unsigned long long* pt_first = nullptr;
  size_t pt_first_cap = 0;
};

std::mutex g_mu;
std::map<std::pair<int, cudaStream_t>, Workspace*> g_ws;

// Frees a workspace (the caller has synchronised its stream).
void free_ws(Workspace* w) {
  void* dev_ptrs[] = {w->counters, w->err, w->ull, w->dbl, w->regs, w->heavy, w->dense, w->csr_dense,
                      w->surv, w->sample_set, w->sample_part, w->stage, w->pt_keys,
                      w->pt_first};
  for (void* p : dev_ptrs)
    if (p) cudaFree(p);
  if (w->host) cudaFreeHost(w->host);
  delete w;
}

int get_ws(cudaStream_t st, Workspace** out) {
  int dev = 0;
  CK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_mu);
  auto key = std::make_pair(dev, st);
  auto it = g_ws.find(key);
  if (it != g_ws.end()) {
    *out = it->second;
    return GM_OK;
  }
  int major = 0;
  CK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
  if (major < 10) return fail(GM_ERR_NO_DEVICE, "device %d is sm_%d0; this library targets sm_100a", dev, major);
  Workspace* w = new Workspace();
  CK(cudaMalloc(&w->counters, 4 * sizeof(int)));
  CK(cudaMalloc(&w->err, sizeof(unsigned long long)));
  CK(cudaMalloc(&w->ull, 4 * sizeof(unsigned long long)));
  CK(cudaMalloc(&w->dbl, 4 * sizeof(double)));
  CK(cudaMallocHost(&w->host, 16 * sizeof(unsigned long long)));
  CK(cudaMemset(w->counters, 0, 4 * sizeof(int)));
  CK(cudaMemset(w->err, 0, sizeof(unsigned long long)));
  CK(cudaDeviceSynchronize());
  g_ws[key] = w;
  *out = w;
  return GM_OK;
}

// Grow a stream-ordered scratch buffer.  The new buffer is allocated before
// the old one is freed, so a failed allocation leaves (*p, *cap) valid.
template <class T>
int grow(T** p, size_t* cap, size_t need, cudaStream_t st, bool zero = false) {
  if (*cap >= need) return GM_OK;
  size_t n = need + need / 4;
  T* q = nullptr;
  CK(cudaMallocAsync((void**)&q, n * sizeof(T), st));
  if (*p) CK(cudaFreeAsync(*p, st));
  *p = q;
  *cap = n;
  if (zero) CK(cudaMemsetAsync(*p, 0, n * sizeof(T), st));
  return GM_OK;
}

int map_device_error(unsigned long long e, unsigned long long vec_base = 0) {
  const int code = (int)(e & 0xFFFFFFFFull);
  const unsigned long long where = (e >> 32) + (code == GM_ERR_EMPTY_VECTOR || code == 3 ? vec_base : 0);
  switch (code) {
    case GM_ERR_EMPTY_VECTOR:
      return fail(code, "EmptyVectorError: vector %llu has no positive entries", where);
    case GM_ERR_INVALID_WEIGHT:
      return fail(code, "InvalidWeightError: weight not finite, > 0 and >= 1e-300 (vector/element %llu)", where);
    case 3:
      return fail(GM_ERR_INVALID_PARAMETER, "InvalidParameterError: vector %llu has more than 2**24 - 4096 elements "
                  "(sketch it with gm_sketch_elements)", where);
    default:
      return fail(code, "device error %d at %llu", code, where);
  }
}

// reads and clears the latched error word; synchronises st
int check_sync(Workspace* ws, cudaStream_t st, unsigned long long vec_base = 0) {
  CK(cudaMemcpyAsync(ws->host, ws->err, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  CK(cudaGetLastError());
  const unsigned long long e = ws->host[0];
  if (e) {
    CK(cudaMemsetAsync(ws->err, 0, sizeof(unsigned long long), st));
    CK(cudaStreamSynchronize(st));
    return map_device_error(e, vec_base);
  }
  return GM_OK;
}

int num_sms() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms > 0 ? sms : 148;
}

// (GM_DEEP_PCT / GM_DRAIN: compile-time overrides for tuning builds only;
// the product build uses the defaults)
#ifndef GM_DEEP_PCT
#define GM_DEEP_PCT 75
#endif
#ifndef GM_DRAIN
#define GM_DRAIN 4
#endif
#ifndef GM_NB
#define GM_NB 16  // lane-table buckets (4 words each)
#endif
#ifndef GM_MINB
#define GM_MINB 2  // resident CTAs per SM the register budget is sized for
#endif
#ifndef GM_VSMALL
#define GM_VSMALL 6
#endif
// k <= 4096: 12-bit lane-table words with a generation tag (no table clear
// per element); larger k: 16-bit words, cleared per element
#ifndef GM_NT
#define GM_NT 256
#endif
#ifndef GM_V
#define GM_V 2
#endif
using CsrDefault = CsrCfg<GM_NT, GM_NB, GM_V, GM_MINB, GM_DEEP_PCT, GM_DRAIN, 12>;
using CsrLargeK = CsrCfg<256, 16, 2, 2, GM_DEEP_PCT, GM_DRAIN, 16>;
// k <= 1024: draw-log lanes (a bit map of drawn positions + the raw draws
// instead of a (position, value) table; gm_csr.cuh).  The lane area shrinks to
// 224 B (k-bit map + 48 logged steps), so two 320-thread CTAs fit per SM (20
// warps instead of 16; 96 registers per thread, no spills), and an element goes
// to the warp walker only when its expected depth reaches the log's capacity
// (measured, config 2: tagged table 0.314 ms; draw log 0.305; with the later
// hand-over 0.3005; with 320 threads 0.296)
#ifndef GM_PB_LOG
#define GM_PB_LOG 10  // (12: the tagged table, for A/B builds)
#endif
#ifndef GM_NT_LOG
#define GM_NT_LOG 320
#endif
#ifndef GM_NB_LOG
#define GM_NB_LOG 12  // logged steps / 4
#endif
#ifndef GM_V_LOG
#define GM_V_LOG GM_V
#endif
#ifndef GM_DEEP_PCT_LOG
#define GM_DEEP_PCT_LOG 100
#endif
using CsrLog = CsrCfg<GM_NT_LOG, GM_NB_LOG, GM_V_LOG, GM_MINB, GM_DEEP_PCT_LOG, GM_DRAIN, GM_PB_LOG>;
// k <= 512: draw-log lanes of 160 B (512-bit map + 48 logged steps) and
// registers of 8 KB per vector leave room for SIX vector slots and 320 threads
// per CTA, two CTAs per SM -- the more vectors a CTA keeps in flight, the fewer
// lanes idle while a slot drains (config 3 per batch: 2 slots 19.4 ms, 4 slots
// 14.6 ms, 5 slots 13.5 ms, 6 slots 12.98 ms; 7 slots x 288 threads 13.27; 8
// slots x 256 threads 13.85)
#ifndef GM_PB_SMALL
#define GM_PB_SMALL 9
#endif
#ifndef GM_NB_SMALL
#define GM_NB_SMALL 12
#endif
#ifndef GM_MINB_SMALL
#define GM_MINB_SMALL GM_MINB
#endif
#ifndef GM_NT_SMALL
#define GM_NT_SMALL 320
#endif
#ifndef GM_DEEP_PCT_SMALL
#define GM_DEEP_PCT_SMALL 100
#endif
using CsrSmallK = CsrCfg<GM_NT_SMALL, GM_NB_SMALL, GM_VSMALL, GM_MINB_SMALL, GM_DEEP_PCT_SMALL, GM_DRAIN, GM_PB_SMALL>;
// One vector under many seeds (GM_FLAG_ONE_VECTOR, k <= 512): every slot
// holds the same vector, so a slot's elements outnumber the lanes and two
// slots keep a 512-thread CTA busy; with few slots, element turnover (the
// ticket scan over the slots) is cheapest (config 1: 0.585 ms with the
// 256-thread / 4-slot configuration -> 0.436 ms; 3 slots 0.459, 4 0.467,
// 6 0.50, 8 0.585)
#ifndef GM_VONE
#define GM_VONE 2
#endif
// (tickets per warp batch: 64 / 128 / 256 = config 1 0.356 / 0.268 / 0.262 ms)
#ifndef GM_WQ_ONE
#define GM_WQ_ONE 256
#endif
#ifndef GM_QCAP_ONE
#define GM_QCAP_ONE 64
#endif
// (draw-log lanes of 128 B -- 512-bit map + 32 logged steps -- leave room for
// 640 threads: config 1 0.293 -> 0.275 ms; 768 threads at 80 registers: 0.312)
#ifndef GM_NT_ONE
#define GM_NT_ONE 640
#endif
#ifndef GM_NB_ONE
#define GM_NB_ONE 8
#endif
#ifndef GM_PB_ONE
#define GM_PB_ONE 9
#endif
using CsrOneVec = CsrCfg<GM_NT_ONE, GM_NB_ONE, GM_VONE, 1, GM_DEEP_PCT_LOG, GM_DRAIN, GM_PB_ONE, GM_WQ_ONE, GM_QCAP_ONE>;

template <class C, class IdT, class WT, bool kCount>
int launch_csr_t(const void* ids, const void* w, const int64_t* offsets, int64_t n_vec, u32 k,
               u64 useed, u64 salt, const u64* vseeds, int one_vec, double* y, u64* s, int64_t* em, Workspace* ws,
               cudaStream_t st, int attempt0) {
  auto kern = csr4_kernel<C, IdT, WT, kCount>;
  const size_t smem = csr_smem_bytes<C>(k);
  int per_sm = 0;
  {
    // occupancy per (kernel, smem) is cached: the launch path stays a
    // memset + two kernel launches
    // (per device: cudaFuncSetAttribute applies to the current device only)
    static std::mutex mu;
    static std::map<std::tuple<int, const void*, size_t>, int> cache;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_tuple(dev, (const void*)kern, smem);
    auto it = cache.find(key);
    if (it == cache.end()) {
      int optin = 0;
      CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
      cudaFuncAttributes fa;
      CK(cudaFuncGetAttributes(&fa, kern));
      const int dyn_max = optin - (int)fa.sharedSizeBytes;
      if (smem <= (size_t)dyn_max) {
        // one limit per function (the device maximum), so launches with a
        // smaller k never lower it under a larger k's requirement
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_max));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::NT, smem));
      }
      it = cache.emplace(key, per_sm).first;
    }
    per_sm = it->second;
  }
  if (per_sm < 1) return -1;  // registers do not fit in shared memory: caller falls back
  int64_t grid = (int64_t)per_sm * num_sms();
  const int64_t need_ctas = (n_vec + C::V - 1) / C::V;
  if (grid > need_ctas) grid = need_ctas;
  // own scratch: the K2 heavy kernel relies on ws->dense staying zeroed
  int rc = grow(&ws->csr_dense, &ws->csr_dense_cap, (size_t)grid * C::NWARP * k, st);
  if (rc) return rc;
  CK(cudaMemsetAsync(ws->counters, 0, sizeof(int), st));
  // the slots compute each vector's weight sum, validate its weights and check
  // the divide range themselves when they load it (no prep launch)
  kern<<<(unsigned)grid, C::NT, smem, st>>>((const IdT*)ids, (const WT*)w, offsets, n_vec, k, useed, salt, vseeds,
                                            one_vec, nullptr, nullptr, y, s, em, ws->counters, ws->csr_dense, ws->err,
                                            attempt0, nullptr);
  CK(cudaGetLastError());
  return GM_OK;
}

template <class C, class IdT, class WT>
int launch_csr(const void* ids, const void* w, const int64_t* offsets, int64_t n_vec, u32 k,
               u64 useed, u64 salt, const u64* vseeds, int one_vec, double* y, u64* s, int64_t* em, Workspace* ws,
               cudaStream_t st, int attempt0) {
  return em ? launch_csr_t<C, IdT, WT, true>(ids, w, offsets, n_vec, k, useed, salt, vseeds, one_vec, y, s, em, ws, st,
                                            attempt0)
            : launch_csr_t<C, IdT, WT, false>(ids, w, offsets, n_vec, k, useed, salt, vseeds, one_vec, y, s, em, ws, st,
                                             attempt0);
}

int check_common(int id_bits, int w_bits, int32_t k) {
  if (id_bits != 32 && id_bits != 64) return fail(GM_ERR_INVALID_PARAMETER, "id_bits must be 32 or 64, got %d", id_bits);
  if (w_bits != 32 && w_bits != 64) return fail(GM_ERR_INVALID_PARAMETER, "w_bits must be 32 or 64, got %d", w_bits);
  if (k < 1) return fail(GM_ERR_INVALID_PARAMETER, "InvalidParameterError: k must be >= 1, got %d", k);
  if (k > GM_K_MAX) return fail(GM_ERR_INVALID_PARAMETER, "k=%d exceeds the supported maximum %d", k, GM_K_MAX);
  return GM_OK;
}

template <class IdT, class WT, class W>
int run_elements(const void* ids, const void* w, int64_t n, u32 k, u64 useed, u64 pseed,
                 uint32_t flags, double* y_io, u64* s_io, int64_t* emitted_out, Workspace* ws,
                 cudaStream_t st, int* unset_async = nullptr) {
  // unset_async != nullptr: one pass, walked at the list bound, enqueued
  // without any host synchronisation; the unset-register count goes to
  // *unset_async (device) when the pass ends (gm_sketch_elements_async)
  int rc = grow(&ws->regs, &ws->regs_cap, (size_t)k, st);
  if (rc) return rc;
  const unsigned rgrid = (k + 255) / 256;
  if (n == 0 || (flags & GM_FLAG_EXHAUSTIVE)) CK(cudaMemsetAsync(ws->ull, 0, 4 * sizeof(unsigned long long), st));
  // fresh registers are initialised by the weight-sample launch when n > 0
  const bool fold_init = n > 0 && !(flags & GM_FLAG_ACCUMULATE);
  if (flags & GM_FLAG_ACCUMULATE) {
    CK(cudaMemsetAsync(ws->counters, 0, 4 * sizeof(int), st));
    load_regs_kernel<<<rgrid, 256, 0, st>>>(ws->regs, k, y_io, s_io, ws->counters + 1);
  } else if (!fold_init) {
    init_regs_kernel<<<rgrid, 256, 0, st>>>(ws->regs, k, ws->counters + 1);
  }
  CK(cudaGetLastError());
  if (n > 0) {
    // blocked weight sample (~2^18 items in 1024 coalesced runs of 256)
    const int sgrid = 1024;
    int64_t sampled = 0;
    for (int64_t b = 0; b < sgrid; ++b) {
      const int64_t lo = b * n / sgrid;
      sampled += std::min<int64_t>(lo + SAMPLE_RUN, (b + 1) * n / sgrid) - lo;
    }
    const u32 tcap = 1u << 20;  // >= 4 x the sample
    if ((rc = grow(&ws->sample_set, &ws->sample_set_cap, (size_t)tcap, st))) return rc;
    CK(cudaMemsetAsync(ws->sample_set, 0xFF, (size_t)tcap * sizeof(unsigned long long), st));
    if ((rc = grow(&ws->sample_part, &ws->sample_part_cap, (size_t)(2 * sgrid), st))) return rc;
    // schedule knobs for tests: scale the first tau, fix the list ratio R
    static const double tau_scale = getenv("GM_ELEM_TAU_SCALE") ? atof(getenv("GM_ELEM_TAU_SCALE")) : 1.0;
    static const double r_fixed = getenv("GM_ELEM_R") ? atof(getenv("GM_ELEM_R")) : 0.0;
    TauArgs targs{ws->dbl, ws->sample_part, sgrid, k, (double)n / (double)std::max<int64_t>(sampled, 1),
                  tau_scale, r_fixed, ws->ull, unset_async ? 1 : 0};
    weight_sample_kernel<IdT, WT><<<sgrid, 256, 0, st>>>((const IdT*)ids, (const WT*)w, n, ws->sample_set, tcap,
                                                         ws->sample_part, fold_init ? ws->regs : nullptr, k,
                                                         ws->counters + 1, targs, (unsigned*)(ws->counters + 3));
    CK(cudaGetLastError());
    const int64_t heavy_need = std::min<int64_t>(n, (int64_t)1 << 22);
    rc = grow(&ws->heavy, &ws->heavy_cap, (size_t)heavy_need, st);
    if (rc) return rc;
    // per-warp dense Fisher-Yates arrays of the heavy walk (k words each); for
    // large k the grid shrinks so the scratch stays <= 1 GB
    const int64_t heavy_blocks = std::max<int64_t>(
        1, std::min<int64_t>((int64_t)num_sms() * 4, ((int64_t)1 << 30) / ((int64_t)NWARP * k * (int64_t)sizeof(W))));
    rc = grow(&ws->dense, &ws->dense_cap, (size_t)heavy_blocks * NWARP * k * (sizeof(W) / 4), st, true);
    if (rc) return rc;
    W* dense = reinterpret_cast<W*>(ws->dense);
    int light_per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&light_per_sm, elem_light_kernel<IdT, WT, W>, NT, 0));
    int64_t lgrid = (int64_t)light_per_sm * num_sms();
    lgrid = std::min<int64_t>(lgrid, (n + NT - 1) / NT);
    // filter pass (HBM-streaming first-arrival test against the list bound
    // tau_hi, survivors compacted into a list)
    // for finite thresholds; a failed pass whose next tau is still <= tau_hi
    // re-walks the list instead of streaming the input again.  The fused light
    // kernel serves tau = +inf, a survivor-list overflow and GM_ELEM_FUSED=1.
    static const bool fused_only = getenv("GM_ELEM_FUSED") && atoi(getenv("GM_ELEM_FUSED")) == 1;
    const int64_t surv_cap = std::min<int64_t>(n, (int64_t)1 << 26);
    if ((rc = grow(&ws->surv, &ws->surv_cap, (size_t)surv_cap, st))) return rc;
    const int64_t fgrid = std::min<int64_t>((n / 4 + 2 * NT - 1) / (2 * NT) + 1, (int64_t)num_sms() * 2 * filter_minb<IdT, WT>());
    int surv_per_sm = 0;  // the list walk is latency-bound: as many resident CTAs as fit
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&surv_per_sm, elem_survivor_kernel<W>, NT, 0));
    surv_per_sm = std::max(surv_per_sm, 1);
    if (unset_async) {  // one pass at the list bound, nothing read back
      elem_filter_kernel<IdT, WT><<<(unsigned)fgrid, NT, 0, st>>>(
          (const IdT*)ids, (const WT*)w, n, k, useed, ws->dbl + 3, ws->surv, surv_cap, ws->ull + 2, nullptr, ws->err);
      elem_survivor_kernel<W><<<(unsigned)(num_sms() * surv_per_sm), NT, 0, st>>>(
          ws->surv, ws->ull + 2, surv_cap, k, useed, pseed, ws->dbl, ws->regs, ws->counters + 1, ws->heavy,
          (int64_t)ws->heavy_cap, ws->ull, nullptr);
      elem_heavy_kernel<IdT, WT, W><<<(unsigned)heavy_blocks, NT, 0, st>>>(
          (const IdT*)ids, (const WT*)w, ws->surv, k, useed, pseed, ws->dbl, ws->regs, ws->counters + 1, ws->heavy,
          ws->ull, (int64_t)ws->heavy_cap, dense, nullptr, (unsigned*)(ws->counters + 2), y_io, s_io);
      CK(cudaGetLastError());
      CK(cudaMemcpyAsync(unset_async, ws->counters + 1, sizeof(int), cudaMemcpyDeviceToDevice, st));
      return GM_OK;
    }
    const double lk = std::log((double)k);
    double tau_h = 0.0, tau_hi_h = 0.0, R = 2.0;
    bool list_ok = false;  // the survivor list holds every element with first arrival <= tau_hi_h
    for (int attempt = 0;; ++attempt) {
      const int att = (flags & GM_FLAG_EXHAUSTIVE) ? 5 : attempt;
      bool rebuild = true;
      if (att >= 5) {  // +inf: full queues (sketch_naive)
        tau_h = tau_hi_h = std::numeric_limits<double>::infinity();
      } else if (attempt > 0) {  // from the unset fraction f: P(unset) = exp(-W tau)
        const int unset = (int)(ws->host[0] & 0xFFFFFFFFull);
        const double f = (double)unset / (double)k;
        const double W_est = f < 1.0 ? -std::log(f) / tau_h : 0.0;
        const double next = W_est > 0.0 ? std::max((lk + 3.0 + 2.0 * attempt) / W_est, 2.0 * tau_h)
                                        : tau_h * (double)k;
        tau_h = next;
        if (list_ok && next <= tau_hi_h) rebuild = false;
        else tau_hi_h = R * next;
      }
      if (att >= 5 || attempt > 0) {
        double* up = reinterpret_cast<double*>(ws->host + 6);
        up[0] = tau_h;
        up[1] = tau_hi_h;
        CK(cudaMemcpyAsync(ws->dbl, up, sizeof(double), cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(ws->dbl + 3, up + 1, sizeof(double), cudaMemcpyHostToDevice, st));
      }  // attempt 0: the sample launch set tau and tau_hi
      if (attempt > 0 || att >= 5) CK(cudaMemsetAsync(ws->ull, 0, sizeof(unsigned long long), st));  // the sample launch clears it at attempt 0
      bool use_filter = !fused_only && att < 4;
      for (int round = 0; round < 2; ++round) {
        if (use_filter) {
          if (rebuild) {
            if (attempt > 0 || att >= 5) CK(cudaMemsetAsync(ws->ull + 2, 0, sizeof(unsigned long long), st));
            elem_filter_kernel<IdT, WT><<<(unsigned)fgrid, NT, 0, st>>>(
                (const IdT*)ids, (const WT*)w, n, k, useed, ws->dbl + 3, ws->surv, surv_cap,
                ws->ull + 2, emitted_out ? ws->ull + 1 : nullptr, ws->err);
            CK(cudaGetLastError());
          }
          elem_survivor_kernel<W><<<(unsigned)(num_sms() * surv_per_sm), NT, 0, st>>>(
              ws->surv, ws->ull + 2, surv_cap, k, useed, pseed, ws->dbl,
              ws->regs, ws->counters + 1, ws->heavy, (int64_t)ws->heavy_cap, ws->ull,
              emitted_out ? ws->ull + 1 : nullptr);
        } else {
          elem_light_kernel<IdT, WT, W><<<(unsigned)lgrid, NT, 0, st>>>(
              (const IdT*)ids, (const WT*)w, n, k, useed, pseed, ws->dbl, ws->regs, ws->counters + 1,
              ws->heavy, (int64_t)ws->heavy_cap, ws->ull, emitted_out ? ws->ull + 1 : nullptr, ws->err);
        }
        CK(cudaGetLastError());
        elem_heavy_kernel<IdT, WT, W><<<(unsigned)heavy_blocks, NT, 0, st>>>(
            (const IdT*)ids, (const WT*)w, use_filter ? ws->surv : nullptr, k, useed, pseed, ws->dbl, ws->regs,
            ws->counters + 1,
            ws->heavy, ws->ull, (int64_t)ws->heavy_cap, dense,
            emitted_out ? ws->ull + 1 : nullptr, (unsigned*)(ws->counters + 2), y_io, s_io);
        // (its last CTA stores the registers: with every attempt, a no-op
        // rewrite when another follows, so a single-attempt call synchronises once)
        CK(cudaGetLastError());
        // accumulate: a loaded register above this pass's tau is not final
        // (counting only unset ones lost arrivals in (tau, y_old))
        if (flags & GM_FLAG_ACCUMULATE) {
          count_unfinished_kernel<<<1, 1024, 0, st>>>(ws->regs, k, ws->dbl, ws->counters + 1);
          CK(cudaGetLastError());
        }
        CK(cudaMemcpyAsync(ws->host, ws->counters + 1, sizeof(int), cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(ws->host + 1, ws->ull, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(ws->host + 3, ws->ull + 2, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(ws->host + 8, ws->err, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        if (emitted_out) CK(cudaMemcpyAsync(ws->host + 2, ws->ull + 1, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        if (attempt == 0 && att < 5) CK(cudaMemcpyAsync(ws->host + 4, ws->dbl, 4 * sizeof(double), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (attempt == 0 && att < 5) {
          const double* d = reinterpret_cast<const double*>(ws->host + 4);
          tau_h = d[0];
          tau_hi_h = d[3];
          R = tau_h > 0.0 ? std::max(2.0, tau_hi_h / tau_h) : 2.0;
        }
        if (use_filter) list_ok = true;
        if (use_filter && (int64_t)ws->host[3] > surv_cap) {  // list overflow: redo the pass fused (idempotent)
          use_filter = false;
          list_ok = false;
          CK(cudaMemsetAsync(ws->ull, 0, sizeof(unsigned long long), st));
          continue;
        }
        break;
      }
      const int unset = (int)(ws->host[0] & 0xFFFFFFFFull);
      const unsigned long long nheavy = ws->host[1];
      if (nheavy > ws->heavy_cap)
        return fail(GM_ERR_CUDA, "internal: heavy-element list overflow (%llu > %zu)", nheavy, ws->heavy_cap);
      if (unset == 0 || ws->host[8] || (flags & GM_FLAG_EXHAUSTIVE) || attempt >= 5) break;
    }
  }
  if (n > 0) {  // the last attempt stored the registers and read the counters back (synchronised)
    CK(cudaGetLastError());
    const unsigned long long e = ws->host[8];
    if (e) {
      CK(cudaMemsetAsync(ws->err, 0, sizeof(unsigned long long), st));
      CK(cudaStreamSynchronize(st));
      return map_device_error(e);
    }
    if (emitted_out) *emitted_out = (int64_t)ws->host[2];
    return GM_OK;
  }
  store_regs_kernel<<<rgrid, 256, 0, st>>>(ws->regs, k, y_io, s_io);
  CK(cudaGetLastError());
  rc = check_sync(ws, st);
  if (rc) return rc;
  CK(cudaMemcpyAsync(ws->host, ws->counters + 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (emitted_out) *emitted_out = 0;
  return GM_OK;
}

// K2 for every id/weight width; queues of more than 65536 customers use
// 64-bit Fisher-Yates words (32-bit positions and values) and exact 64-bit draws
int dispatch_elements(const void* ids, int id_bits, const void* w, int w_bits, int64_t n, u32 k, u64 useed,
                      u64 pseed, uint32_t flags, double* y_io, u64* s_io, int64_t* emitted_out, Workspace* ws,
                      cudaStream_t st, int* unset_async) {
#define GM_ELEM_RUN(I, F, W) \
  return run_elements<I, F, W>(ids, w, n, k, useed, pseed, flags, y_io, s_io, emitted_out, ws, st, unset_async)
  if (k <= 65536u) {
    if (id_bits == 32 && w_bits == 32) GM_ELEM_RUN(u32, float, u32);
    if (id_bits == 32) GM_ELEM_RUN(u32, double, u32);
    if (w_bits == 32) GM_ELEM_RUN(u64, float, u32);
    GM_ELEM_RUN(u64, double, u32);
  }
  if (id_bits == 32 && w_bits == 32) GM_ELEM_RUN(u32, float, u64);
  if (id_bits == 32) GM_ELEM_RUN(u32, double, u64);
  if (w_bits == 32) GM_ELEM_RUN(u64, float, u64);
  GM_ELEM_RUN(u64, double, u64);
#undef GM_ELEM_RUN
}

}  // namespace

extern "C" {

int gm_version(void) { return 100; }

int gm_debug_error(unsigned long long* out) {
#ifdef GM_DEBUG
  CK(cudaMemcpyFromSymbol(out, g_dbg_err, sizeof(unsigned long long)));
  return GM_OK;
#else
  *out = 0;
  return GM_OK;
#endif
}

const char* gm_last_error(void) { return g_msg; }

// GM_STATS builds only (tools/stats.py): read and clear the 16 work counters
int gm_stats_read(unsigned long long* out16) {
#ifdef GM_STATS
  CK(cudaMemcpyFromSymbol(out16, g_stats, sizeof(unsigned long long) * 16));
  unsigned long long z[16] = {0};
  CK(cudaMemcpyToSymbol(g_stats, z, sizeof(z)));
  return GM_OK;
#else
  (void)out16;
  return fail(GM_ERR_INVALID_PARAMETER, "library built without GM_STATS");
#endif
}

int gm_check_pairs(const void* ids, int id_bits, const void* w, int w_bits, int64_t n, int64_t* first_bad,
                   int64_t* first_conflict, void* uniq_ids, void* uniq_w, int64_t* n_uniq, void* stream) {
  g_msg[0] = 0;
  (void)cudaGetLastError();
  if ((id_bits != 32 && id_bits != 64) || (w_bits != 32 && w_bits != 64) || n < 0)
    return fail(GM_ERR_INVALID_PARAMETER, "gm_check_pairs: bad id_bits/w_bits/n");
  if ((uniq_ids == nullptr) != (uniq_w == nullptr))
    return fail(GM_ERR_INVALID_PARAMETER, "gm_check_pairs: uniq_ids and uniq_w go together");
  *first_bad = *first_conflict = -1;
  if (n_uniq) *n_uniq = 0;
  if (n == 0) return GM_OK;
  cudaStream_t st = (cudaStream_t)stream;
  Workspace* ws = nullptr;
  int rc = get_ws(st, &ws);
  if (rc) return rc;
  size_t cap = 1024;
  while (cap < 2 * (size_t)n) cap <<= 1;
  if ((rc = grow(&ws->pt_keys, &ws->pt_keys_cap, cap + 1, st))) return rc;
  if ((rc = grow(&ws->pt_first, &ws->pt_first_cap, cap + 1, st))) return rc;
  CK(cudaMemsetAsync(ws->pt_keys, 0xFF, (cap + 1) * sizeof(u64), st));
  CK(cudaMemsetAsync(ws->pt_first, 0xFF, (cap + 1) * sizeof(unsigned long long), st));
  CK(cudaMemsetAsync(ws->ull, 0xFF, 2 * sizeof(unsigned long long), st));
  CK(cudaMemsetAsync(ws->ull + 2, 0, sizeof(unsigned long long), st));
  const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 8);
  const u64 mask = cap - 1;
#define GM_PAIRS(I, W)                                                                                        \
  do {                                                                                                        \
    pairs_insert_kernel<I><<<grid, 256, 0, st>>>((const I*)ids, n, ws->pt_keys, ws->pt_first, mask);          \
    pairs_check_kernel<I, W><<<grid, 256, 0, st>>>((const I*)ids, (const W*)w, n, ws->pt_keys, ws->pt_first, \
                                                   mask, ws->ull, (I*)uniq_ids, (W*)uniq_w);                  \
  } while (0)
  if (id_bits == 32 && w_bits == 32) GM_PAIRS(u32, float);
  else if (id_bits == 32) GM_PAIRS(u32, double);
  else if (w_bits == 32) GM_PAIRS(u64, float);
  else GM_PAIRS(u64, double);
#undef GM_PAIRS
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(ws->host, ws->ull, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  *first_bad = ws->host[0] == ~0ull ? -1 : (int64_t)ws->host[0];
  *first_conflict = ws->host[1] == ~0ull ? -1 : (int64_t)ws->host[1];
  if (n_uniq) *n_uniq = (int64_t)ws->host[2];
  return GM_OK;
}

// -DGM_EVENTS builds only (tools/timeline.py): slot events (n x 2 u64, up
// to 32768) and their count; clears them
int gm_trace_read(unsigned long long* ev_out, unsigned* n_out) {
#ifdef GM_EVENTS
  CK(cudaDeviceSynchronize());
  unsigned n = 0;
  CK(cudaMemcpyFromSymbol(&n, g_trace_n, sizeof(n)));
  if (n > 32768) n = 32768;
  if (n) CK(cudaMemcpyFromSymbol(ev_out, g_trace, sizeof(unsigned long long) * 2 * n));
  *n_out = n;
  unsigned zn = 0;
  CK(cudaMemcpyToSymbol(g_trace_n, &zn, sizeof(zn)));
  return GM_OK;
#else
  (void)ev_out;
  (void)n_out;
  return fail(GM_ERR_INVALID_PARAMETER, "library built without GM_EVENTS");
#endif
}

// Lifecycle: scratch is created lazily per (device, stream) by the first
// call on that stream and kept for the stream's next calls.
int gm_release_stream(void* stream) {
  g_msg[0] = 0;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  Workspace* w = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_ws.find(std::make_pair(dev, (cudaStream_t)stream));
    if (it == g_ws.end()) return GM_OK;
    w = it->second;
    g_ws.erase(it);
  }
  CK(cudaStreamSynchronize((cudaStream_t)stream));
  free_ws(w);
  CK(cudaGetLastError());
  return GM_OK;
}

int gm_finalize(void) {
  g_msg[0] = 0;
  std::map<std::pair<int, cudaStream_t>, Workspace*> all;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    all.swap(g_ws);
  }
  int cur = 0;
  CK(cudaGetDevice(&cur));
  for (auto& kv : all) {
    CK(cudaSetDevice(kv.first.first));
    CK(cudaDeviceSynchronize());
    free_ws(kv.second);
  }
  CK(cudaSetDevice(cur));
  return GM_OK;
}

int gm_workspace_count(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  return (int)g_ws.size();
}

// ---- NCCL register exchange (gm_comm.cuh) ----
#define NK(call)                                                                                     \
  do {                                                                                               \
    ncclResult_t r_ = (call);                                                                        \
    if (r_ != ncclSuccess) return fail(GM_ERR_COMM, "%s failed: %s", #call, nccl_api().error_string(r_)); \
  } while (0)

static int comm_api_ok() {
  NcclApi& a = nccl_api();
  return a.ok ? GM_OK : fail(GM_ERR_COMM, "%s", a.why);
}

int gm_comm_unique_id(void* id_out) {
  g_msg[0] = 0;
  int rc = comm_api_ok();
  if (rc) return rc;
  if (!id_out) return fail(GM_ERR_INVALID_PARAMETER, "id_out is NULL");
  ncclUniqueId id;
  NK(nccl_api().get_unique_id(&id));
  memcpy(id_out, &id, sizeof(id));
  return GM_OK;
}

int gm_comm_id_bytes(void) { return (int)sizeof(ncclUniqueId); }

int gm_comm_init(const void* id, int nranks, int rank, void** comm_out) {
  g_msg[0] = 0;
  int rc = comm_api_ok();
  if (rc) return rc;
  if (!id || !comm_out || nranks < 1 || rank < 0 || rank >= nranks)
    return fail(GM_ERR_INVALID_PARAMETER, "gm_comm_init: bad arguments (nranks %d, rank %d)", nranks, rank);
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  GmComm* c = new GmComm();
  CK(cudaGetDevice(&c->device));
  c->nranks = nranks;
  c->rank = rank;
  const ncclResult_t r = nccl_api().comm_init_rank(&c->comm, nranks, uid, rank);
  if (r != ncclSuccess) {
    delete c;
    return fail(GM_ERR_COMM, "ncclCommInitRank failed: %s", nccl_api().error_string(r));
  }
  *comm_out = c;
  return GM_OK;
}

int gm_comm_destroy(void* comm) {
  g_msg[0] = 0;
  if (!comm) return GM_OK;
  GmComm* c = (GmComm*)comm;
  if (c->ybuf) cudaFree(c->ybuf);
  if (c->sbuf) cudaFree(c->sbuf);
  if (c->comm && nccl_api().ok) NK(nccl_api().comm_destroy(c->comm));
  delete c;
  return GM_OK;
}

static int comm_scratch(GmComm* c, size_t regs) {
  if (c->cap >= regs) return GM_OK;
  if (c->ybuf) CK(cudaFree(c->ybuf));
  if (c->sbuf) CK(cudaFree(c->sbuf));
  c->ybuf = nullptr;
  c->sbuf = nullptr;
  c->cap = 0;
  CK(cudaMalloc(&c->ybuf, regs * sizeof(double)));
  CK(cudaMalloc(&c->sbuf, regs * sizeof(u64)));
  c->cap = regs;
  return GM_OK;
}

int gm_allreduce_min_registers(void* comm, double* y, uint64_t* s, int32_t k, void* stream) {
  g_msg[0] = 0;
  (void)cudaGetLastError();
  int rc = comm_api_ok();
  if (rc) return rc;
  if (!comm || k < 1) return fail(GM_ERR_INVALID_PARAMETER, "gm_allreduce_min_registers: bad arguments");
  GmComm* c = (GmComm*)comm;
  cudaStream_t st = (cudaStream_t)stream;
  if ((rc = comm_scratch(c, (size_t)k))) return rc;
  NK(nccl_api().all_reduce(y, c->ybuf, (size_t)k, ncclFloat64, ncclMin, c->comm, st));
  mask_min_ids_kernel<<<(unsigned)std::min<int64_t>(((int64_t)k + 255) / 256, 1024), 256, 0, st>>>(y, c->ybuf, s,
                                                                                                   c->sbuf, (u32)k);
  CK(cudaGetLastError());
  NK(nccl_api().all_reduce(c->sbuf, s, (size_t)k, ncclUint64, ncclMin, c->comm, st));
  CK(cudaMemcpyAsync(y, c->ybuf, (size_t)k * sizeof(double), cudaMemcpyDeviceToDevice, st));
  return GM_OK;
}

int gm_allgather_merge_registers(void* comm, double* y, uint64_t* s, int32_t k, void* stream) {
  g_msg[0] = 0;
  (void)cudaGetLastError();
  int rc = comm_api_ok();
  if (rc) return rc;
  if (!comm || k < 1) return fail(GM_ERR_INVALID_PARAMETER, "gm_allgather_merge_registers: bad arguments");
  GmComm* c = (GmComm*)comm;
  cudaStream_t st = (cudaStream_t)stream;
  if ((rc = comm_scratch(c, (size_t)k * c->nranks))) return rc;
  NK(nccl_api().group_start());
  NK(nccl_api().all_gather(y, c->ybuf, (size_t)k, ncclFloat64, c->comm, st));
  NK(nccl_api().all_gather(s, c->sbuf, (size_t)k, ncclUint64, c->comm, st));
  NK(nccl_api().group_end());
  const unsigned grid = (unsigned)std::min<int64_t>(((int64_t)k + 255) / 256, 4096);
  merge_kernel<<<grid, 256, 0, st>>>(c->ybuf, c->sbuf, c->nranks, (u32)k, y, s);
  CK(cudaGetLastError());
  return GM_OK;
}

int gm_stream_status(void* stream) {
  Workspace* ws = nullptr;
  int rc = get_ws((cudaStream_t)stream, &ws);
  if (rc) return rc;
  return check_sync(ws, (cudaStream_t)stream);
}

int gm_sketch_elements(const void* ids, int id_bits, const void* w, int w_bits, int64_t n,
                       int32_t k, uint64_t global_seed, uint64_t stream_salt, uint32_t flags,
                       double* y_io, uint64_t* s_io, int64_t* emitted_out, void* stream);

// k too large for shared-memory registers: one grid-wide sketch per vector
static int csr_by_elements(const void* ids, int id_bits, const void* w, int w_bits,
                           const int64_t* offsets, int64_t n_vec, int32_t k, uint64_t seed,
                           uint64_t salt, uint32_t flags, double* y_out, uint64_t* s_out,
                           int64_t* emitted_out, cudaStream_t st) {
  int64_t* off = (int64_t*)malloc((size_t)(n_vec + 1) * 8);
  if (!off) return fail(GM_ERR_CUDA, "host allocation failed");
  cudaError_t e = cudaMemcpyAsync(off, offsets, (size_t)(n_vec + 1) * 8, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    free(off);
    return fail(GM_ERR_CUDA, "offsets readback failed: %s", cudaGetErrorString(e));
  }
  int rc = GM_OK;
  for (int64_t v = 0; v < n_vec && rc == GM_OK; ++v) {
    const int64_t lo = off[v], n = off[v + 1] - lo;
    if (n == 0) {
      rc = fail(GM_ERR_EMPTY_VECTOR, "EmptyVectorError: vector %lld has no positive entries", (long long)v);
      break;
    }
    int64_t em = 0;
    rc = gm_sketch_elements((const char*)ids + lo * (id_bits / 8), id_bits,
                            (const char*)w + lo * (w_bits / 8), w_bits, n, k, seed, salt,
                            flags & GM_FLAG_EXHAUSTIVE, y_out + v * (int64_t)k, s_out + v * (int64_t)k,
                            emitted_out ? &em : nullptr, st);
    if (rc == GM_OK && emitted_out) {
      cudaError_t e2 = cudaMemcpyAsync(emitted_out + v, &em, 8, cudaMemcpyHostToDevice, st);
      if (e2 == cudaSuccess) e2 = cudaStreamSynchronize(st);
      if (e2 != cudaSuccess) rc = fail(GM_ERR_CUDA, "%s", cudaGetErrorString(e2));
    }
  }
  free(off);
  return rc;
}

// The batched K1 launch (csr4_kernel) for every id/weight width; vseeds
// (device, nullable): per-vector global seeds.
static int csr_dispatch(const void* ids, int id_bits, const void* w, int w_bits, const int64_t* offsets,
                        int64_t n_vec, int32_t k, uint64_t global_seed, uint64_t stream_salt, const uint64_t* vseeds,
                        uint32_t flags, double* y_out, uint64_t* s_out, int64_t* emitted_out, cudaStream_t st) {
  int rc = check_common(id_bits, w_bits, k);
  if (rc) return rc;
  if (n_vec < 0) return fail(GM_ERR_INVALID_PARAMETER, "n_vec must be >= 0");
  if (n_vec == 0) return GM_OK;
  Workspace* ws = nullptr;
  rc = get_ws(st, &ws);
  if (rc) return rc;
  const u64 useed = global_seed, salt = stream_salt;
  const u32 kk = (u32)k;
  const bool small_k = kk <= 512;  // CsrSmallK: four vector slots
  const int one_vec = (flags & GM_FLAG_ONE_VECTOR) ? 1 : 0;
  if (one_vec && !vseeds) return fail(GM_ERR_INVALID_PARAMETER, "GM_FLAG_ONE_VECTOR needs per-sketch seeds");
  // exhaustive = a single pass with tau = +inf (pass_tau's last attempt)
  const int a0 = (flags & GM_FLAG_EXHAUSTIVE) ? 3 : 0;
#define GM_CSR_LAUNCH(I, W)                                                                                          \
  rc = one_vec && kk <= 512                                                                                    \
           ? launch_csr<CsrOneVec, I, W>(ids, w, offsets, n_vec, kk, useed, salt, vseeds, one_vec, y_out, s_out,   \
                                         emitted_out, ws, st, a0)                                                    \
       : small_k ? launch_csr<CsrSmallK, I, W>(ids, w, offsets, n_vec, kk, useed, salt, vseeds, one_vec, y_out,     \
                                             s_out, emitted_out, ws, st, a0)                                         \
       : kk <= 1024                                                                                                  \
           ? launch_csr<CsrLog, I, W>(ids, w, offsets, n_vec, kk, useed, salt, vseeds, one_vec, y_out, s_out,       \
                                      emitted_out, ws, st, a0)                                                       \
       : kk <= CsrDefault::KMAX                                                                                      \
           ? launch_csr<CsrDefault, I, W>(ids, w, offsets, n_vec, kk, useed, salt, vseeds, one_vec, y_out, s_out,   \
                                          emitted_out, ws, st, a0)                                                   \
           : launch_csr<CsrLargeK, I, W>(ids, w, offsets, n_vec, kk, useed, salt, vseeds, one_vec, y_out, s_out,    \
                                         emitted_out, ws, st, a0)
  if (id_bits == 32 && w_bits == 32) GM_CSR_LAUNCH(u32, float);
  else if (id_bits == 32) GM_CSR_LAUNCH(u32, double);
  else if (w_bits == 32) GM_CSR_LAUNCH(u64, float);
  else GM_CSR_LAUNCH(u64, double);
#undef GM_CSR_LAUNCH
  if (rc == -1) {
    if (vseeds) return fail(GM_ERR_INVALID_PARAMETER, "per-sketch seeds need k small enough for shared-memory registers");
    return csr_by_elements(ids, id_bits, w, w_bits, offsets, n_vec, k, global_seed, stream_salt, flags, y_out, s_out,
                           emitted_out, st);
  }
  if (rc) return rc;
  if (flags & GM_FLAG_ASYNC) return GM_OK;
  return check_sync(ws, st);
}

int gm_sketch_csr(const void* ids, int id_bits, const void* w, int w_bits, const int64_t* offsets,
                  int64_t n_vec, int32_t k, uint64_t global_seed, uint64_t stream_salt,
                  uint32_t flags, double* y_out, uint64_t* s_out, int64_t* emitted_out,
                  void* stream) {
  g_msg[0] = 0;
  (void)cudaGetLastError();
  return csr_dispatch(ids, id_bits, w, w_bits, offsets, n_vec, k, global_seed, stream_salt, nullptr, flags, y_out,
                      s_out, emitted_out, (cudaStream_t)stream);
}

int gm_sketch_csr_seeded(const void* ids, int id_bits, const void* w, int w_bits, const int64_t* offsets,
                         int64_t n_vec, int32_t k, const uint64_t* global_seeds, uint64_t stream_salt,
                         uint32_t flags, double* y_out, uint64_t* s_out, int64_t* emitted_out, void* stream) {
  g_msg[0] = 0;
  (void)cudaGetLastError();
  if (!global_seeds) return fail(GM_ERR_INVALID_PARAMETER, "global_seeds must be a device array of n_vec seeds");
  return csr_dispatch(ids, id_bits, w, w_bits, offsets, n_vec, k, 0, stream_salt, global_seeds, flags, y_out, s_out,
                      emitted_out, (cudaStream_t)stream);
}

// One vector alone is sketched by the grid-wide kernels (K2: weight sample,
// filter, list walk, heavy walk -- every SM) once it has this many elements;
// below it the batched kernel's single CTA is faster (GM_SINGLE_GRID_MIN
// overrides; 0 disables).  Results are identical (ids are distinct within a
// vector, so K2's duplicate rule never applies).
static int64_t single_vector_grid_min() {
  static const int64_t v = getenv("GM_SINGLE_GRID_MIN") ? atoll(getenv("GM_SINGLE_GRID_MIN")) : 4096;
  return v > 0 ? v : INT64_MAX;
}

static int single_vector_grid(const void* ids, int id_bits, const void* w, int w_bits, int64_t n, int32_t k,
                              uint64_t seed, uint64_t salt, uint32_t flags, double* y_out, uint64_t* s_out,
                              int64_t* emitted_out, Workspace* ws, cudaStream_t st) {
  const size_t ib = (size_t)n * (id_bits / 8), wb = (size_t)n * (w_bits / 8), yb = (size_t)k * 8;
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  const bool s32 = flags & GM_FLAG_S32;
  int rc = grow((unsigned char**)&ws->stage, &ws->stage_cap, al(ib) + al(wb) + 2 * al(yb) + al(yb / 2), st);
  if (rc) return rc;
  unsigned char* base = (unsigned char*)ws->stage;
  void* d_ids = base;
  void* d_w = base + al(ib);
  double* d_y = (double*)(base + al(ib) + al(wb));
  u64* d_s = (u64*)((unsigned char*)d_y + al(yb));
  u32* d_s32 = (u32*)((unsigned char*)d_s + al(yb));
  CK(cudaMemcpyAsync(d_ids, ids, ib, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_w, w, wb, cudaMemcpyHostToDevice, st));
  rc = gm_sketch_elements(d_ids, id_bits, d_w, w_bits, n, k, seed, salt, flags & GM_FLAG_EXHAUSTIVE, d_y, d_s,
                          emitted_out, st);
  if (rc) return rc;
  CK(cudaMemcpyAsync(y_out, d_y, yb, cudaMemcpyDeviceToHost, st));
  if (s32) {
    narrow_u32_kernel<<<(unsigned)((k + 255) / 256), 256, 0, st>>>(d_s, d_s32, k);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(s_out, d_s32, yb / 2, cudaMemcpyDeviceToHost, st));
  } else {
    CK(cudaMemcpyAsync(s_out, d_s, yb, cudaMemcpyDeviceToHost, st));
  }
  CK(cudaStreamSynchronize(st));
  return GM_OK;
}

// device address of a page-locked host buffer (nullptr if the buffer is
// pageable): the kernels can store their results straight into it
static void* pinned_device_ptr(void* host) {
  if (!host) return nullptr;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, host) != cudaSuccess) {
    (void)cudaGetLastError();
    return nullptr;
  }
  return a.type == cudaMemoryTypeHost ? a.devicePointer : nullptr;
}

int gm_sketch_csr_host(const void* ids, int id_bits, const void* w, int w_bits,
                       const int64_t* offsets, int64_t n_vec, int32_t k, uint64_t global_seed,
                       uint64_t stream_salt, uint32_t flags, double* y_out, uint64_t* s_out,
                       int64_t* emitted_out, void* stream) {
  g_msg[0] = 0;
  (void)cudaGetLastError();
  int rc = check_common(id_bits, w_bits, k);
  if (rc) return rc;
  if (n_vec < 0) return fail(GM_ERR_INVALID_PARAMETER, "n_vec must be >= 0");
  if (n_vec == 0) return GM_OK;
  cudaStream_t st = (cudaStream_t)stream;
  Workspace* ws = nullptr;
  rc = get_ws(st, &ws);
  if (rc) return rc;
  const bool s32 = flags & GM_FLAG_S32;
  if (s32 && id_bits != 32) return fail(GM_ERR_INVALID_PARAMETER, "GM_FLAG_S32 needs 32-bit ids");
  const int64_t n = offsets[n_vec];
  if (n_vec == 1 && !(flags & GM_FLAG_ASYNC) && offsets[0] == 0 && n >= single_vector_grid_min())
    return single_vector_grid(ids, id_bits, w, w_bits, n, k, global_seed, stream_salt, flags, y_out, s_out,
                              emitted_out, ws, st);
  const size_t ib = (size_t)n * (id_bits / 8), wb = (size_t)n * (w_bits / 8);
  const size_t ob = (size_t)(n_vec + 1) * 8, yb = (size_t)n_vec * k * 8;
  // results go straight to page-locked host buffers (the kernel's stores
  // overlap its compute); pageable ones are staged on the device and copied.
  // GM_FLAG_S32: s is delivered as uint32 (ids are 32-bit), narrowed on the
  // device, so the host receives 12 instead of 16 bytes per register.
  double* dy_host = (double*)pinned_device_ptr(y_out);
  void* ds_host = pinned_device_ptr(s_out);
  int64_t* dem_host = (int64_t*)pinned_device_ptr(emitted_out);
  // A synchronous call has the kernel store into page-locked outputs (the
  // stores overlap its compute); a GM_FLAG_ASYNC call (a stream of batches)
  // stages on the device and lets the copy engine move the registers, which
  // overlaps the next batches' kernels instead of holding their SMs on bus
  // writes (tools/e2e_variants.py).  GM_HOST_ZEROCOPY_OUT: 0 never, 2 always.
  static const int zc_out = getenv("GM_HOST_ZEROCOPY_OUT") ? atoi(getenv("GM_HOST_ZEROCOPY_OUT")) : 1;
  const bool zc = zc_out == 2 || (zc_out == 1 && !(flags & GM_FLAG_ASYNC));
  const bool direct = zc && dy_host && ds_host && (!emitted_out || dem_host);
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  const size_t sb32 = (size_t)n_vec * k * 4;
  const size_t need = al(ib) + al(wb) + al(ob) + (direct ? 0 : al(yb) + al((size_t)n_vec * 8)) +
                      ((!direct || s32) ? al(yb) : 0) + ((s32 && !direct) ? al(sb32) : 0);
  rc = grow((unsigned char**)&ws->stage, &ws->stage_cap, need, st);
  if (rc) return rc;
  unsigned char* p = (unsigned char*)ws->stage;
  auto take = [&](size_t bytes) {
    unsigned char* q = p;
    p += al(bytes);
    return q;
  };
  void* d_ids = take(ib);
  void* d_w = take(wb);
  int64_t* d_off = (int64_t*)take(ob);
  double* d_y = direct ? dy_host : (double*)take(yb);
  u64* d_s = (direct && !s32) ? (u64*)ds_host : (u64*)take(yb);
  int64_t* d_em = !emitted_out ? nullptr : direct ? dem_host : (int64_t*)take((size_t)n_vec * 8);
  u32* d_s32 = !s32 ? nullptr : direct ? (u32*)ds_host : (u32*)take(sb32);
  CK(cudaMemcpyAsync(d_off, offsets, ob, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_w, w, wb, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_ids, ids, ib, cudaMemcpyHostToDevice, st));
  rc = gm_sketch_csr(d_ids, id_bits, d_w, w_bits, d_off, n_vec, k, global_seed, stream_salt,
                     (flags & ~GM_FLAG_S32) | GM_FLAG_ASYNC, d_y, d_s, d_em, stream);
  if (rc) return rc;
  if (s32) {
    const int64_t nr = n_vec * (int64_t)k;
    narrow_u32_kernel<<<(unsigned)std::min<int64_t>((nr + 255) / 256, (int64_t)num_sms() * 8), 256, 0, st>>>(
        d_s, d_s32, nr);
    CK(cudaGetLastError());
  }
  if (!direct) {
    CK(cudaMemcpyAsync(y_out, d_y, yb, cudaMemcpyDeviceToHost, st));
    if (s32) CK(cudaMemcpyAsync(s_out, d_s32, sb32, cudaMemcpyDeviceToHost, st));
    else CK(cudaMemcpyAsync(s_out, d_s, yb, cudaMemcpyDeviceToHost, st));
    if (d_em) CK(cudaMemcpyAsync(emitted_out, d_em, (size_t)n_vec * 8, cudaMemcpyDeviceToHost, st));
  }
  // GM_FLAG_ASYNC: enqueue only (inputs and outputs stay in use until the
  // stream is synchronised; data errors via gm_stream_status)
  if (flags & GM_FLAG_ASYNC) return GM_OK;
  return check_sync(ws, st);
}

int gm_sketch_elements(const void* ids, int id_bits, const void* w, int w_bits, int64_t n,
                       int32_t k, uint64_t global_seed, uint64_t stream_salt, uint32_t flags,
                       double* y_io, uint64_t* s_io, int64_t* emitted_out, void* stream) {
  g_msg[0] = 0;
  (void)cudaGetLastError();
  int rc = check_common(id_bits, w_bits, k);
  if (rc) return rc;
  if (n < 0) return fail(GM_ERR_INVALID_PARAMETER, "n must be >= 0");
  cudaStream_t st = (cudaStream_t)stream;
  Workspace* ws = nullptr;
  rc = get_ws(st, &ws);
  if (rc) return rc;
  const u64 useed = global_seed, pseed = global_seed ^ stream_salt;
  const u32 kk = (u32)k;
  rc = dispatch_elements(ids, id_bits, w, w_bits, n, kk, useed, pseed, flags, y_io, s_io, emitted_out, ws, st,
                         nullptr);
  if (rc) return rc;
  const int unset = (int)(ws->host[0] & 0xFFFFFFFFull);
  if (unset > 0)
    return fail(GM_ERR_INCOMPLETE, "IncompleteSketchError: %d register(s) unset", unset);
  return GM_OK;
}

int gm_sketch_elements_async(const void* ids, int id_bits, const void* w, int w_bits, int64_t n,
                             int32_t k, uint64_t global_seed, uint64_t stream_salt, uint32_t flags,
                             double* y_io, uint64_t* s_io, int32_t* unset_out, void* stream) {
  g_msg[0] = 0;
  (void)cudaGetLastError();
  int rc = check_common(id_bits, w_bits, k);
  if (rc) return rc;
  if (n < 1) return fail(GM_ERR_INVALID_PARAMETER, "gm_sketch_elements_async needs n >= 1");
  if (!unset_out) return fail(GM_ERR_INVALID_PARAMETER, "unset_out must be a device int");
  if (flags & (GM_FLAG_EXHAUSTIVE | GM_FLAG_ACCUMULATE))
    return fail(GM_ERR_INVALID_PARAMETER, "GM_FLAG_EXHAUSTIVE / GM_FLAG_ACCUMULATE need gm_sketch_elements");
  cudaStream_t st = (cudaStream_t)stream;
  Workspace* ws = nullptr;
  rc = get_ws(st, &ws);
  if (rc) return rc;
  const u64 useed = global_seed, pseed = global_seed ^ stream_salt;
  const u32 kk = (u32)k;
  return dispatch_elements(ids, id_bits, w, w_bits, n, kk, useed, pseed, flags, y_io, s_io, nullptr, ws, st,
                           unset_out);
}

int gm_sketch_elements_host(const void* ids, int id_bits, const void* w, int w_bits, int64_t n,
                            int32_t k, uint64_t global_seed, uint64_t stream_salt,
                            uint32_t flags, double* y_io, uint64_t* s_io, int64_t* emitted_out,
                            void* stream) {
  g_msg[0] = 0;
  (void)cudaGetLastError();
  int rc = check_common(id_bits, w_bits, k);
  if (rc) return rc;
  if (n < 0) return fail(GM_ERR_INVALID_PARAMETER, "n must be >= 0");
  cudaStream_t st = (cudaStream_t)stream;
  Workspace* ws = nullptr;
  rc = get_ws(st, &ws);
  if (rc) return rc;
  const size_t ib = (size_t)n * (id_bits / 8), wb = (size_t)n * (w_bits / 8), yb = (size_t)k * 8;
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  rc = grow((unsigned char**)&ws->stage, &ws->stage_cap, al(ib) + al(wb) + 2 * al(yb), st);
  if (rc) return rc;
  unsigned char* base = (unsigned char*)ws->stage;
  void* d_ids = base;
  void* d_w = base + al(ib);
  double* d_y = (double*)(base + al(ib) + al(wb));
  u64* d_s = (u64*)((unsigned char*)d_y + al(yb));
  if (n) {
    CK(cudaMemcpyAsync(d_ids, ids, ib, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_w, w, wb, cudaMemcpyHostToDevice, st));
  }
  if (flags & GM_FLAG_ACCUMULATE) {
    CK(cudaMemcpyAsync(d_y, y_io, yb, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_s, s_io, yb, cudaMemcpyHostToDevice, st));
  }
  rc = gm_sketch_elements(d_ids, id_bits, d_w, w_bits, n, k, global_seed, stream_salt, flags, d_y,
                          d_s, emitted_out, stream);
  if (rc && rc != GM_ERR_INCOMPLETE) return rc;
  CK(cudaMemcpyAsync(y_io, d_y, yb, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(s_io, d_s, yb, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return rc;
}

int gm_merge(const double* y_in, const uint64_t* s_in, int64_t n_sk, int32_t k, double* y_out,
             uint64_t* s_out, void* stream) {
  g_msg[0] = 0;
  (void)cudaGetLastError();
  if (n_sk < 1) return fail(GM_ERR_MISMATCHED, "MismatchedSketchError: cannot merge an empty list of sketches");
  if (k < 1) return fail(GM_ERR_INVALID_PARAMETER, "k must be >= 1");
  const unsigned grid = (unsigned)std::min<int64_t>(((int64_t)k + 255) / 256, 4096);
  merge_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(y_in, s_in, n_sk, (u32)k, y_out, s_out);
  CK(cudaGetLastError());
  return GM_OK;
}

int gm_match_count(const uint64_t* s_a, const uint64_t* s_b, int64_t n_pairs, int32_t k,
                   int32_t* matches, void* stream) {
  g_msg[0] = 0;
  (void)cudaGetLastError();
  if (k < 1) return fail(GM_ERR_INVALID_PARAMETER, "k must be >= 1");
  if (n_pairs <= 0) return GM_OK;
  match_count_kernel<<<(unsigned)n_pairs, 256, 0, (cudaStream_t)stream>>>(s_a, s_b, n_pairs, (u32)k, matches);
  CK(cudaGetLastError());
  return GM_OK;
}

int gm_cardinality(const double* y, int64_t n_sk, int32_t k, double* sum_out, double* card_out, void* stream) {
  g_msg[0] = 0;
  (void)cudaGetLastError();
  if (k < 1) return fail(GM_ERR_INVALID_PARAMETER, "k must be >= 1");
  if (n_sk <= 0) return GM_OK;
  exact_sum_kernel<<<(unsigned)n_sk, 256, 0, (cudaStream_t)stream>>>(y, n_sk, (u32)k, sum_out, card_out);
  CK(cudaGetLastError());
  return GM_OK;
}

int gm_uniform_open_batch(const uint64_t* global_seeds, const uint64_t* elements,
                          const uint64_t* steps, int64_t n, double* out, void* stream) {
  g_msg[0] = 0;
  (void)cudaGetLastError();
  if (n <= 0) return GM_OK;
  uniform_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(global_seeds, elements, steps, n, out);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize((cudaStream_t)stream));
  return GM_OK;
}

int gm_perm_draw_batch(const uint64_t* perm_seeds, const uint64_t* elements, const uint64_t* steps,
                       const uint32_t* ks, int64_t n, uint32_t* out, void* stream) {
  g_msg[0] = 0;
  (void)cudaGetLastError();
  if (n <= 0) return GM_OK;
  randint_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(perm_seeds, elements, steps, ks, n, out);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize((cudaStream_t)stream));
  return GM_OK;
}

int gm_rand_int_between_batch(const uint64_t* perm_seeds, const uint64_t* elements, const uint64_t* steps,
                              const uint64_t* m_minus_1, int64_t n, uint64_t* out, void* stream) {
  g_msg[0] = 0;
  (void)cudaGetLastError();
  if (n <= 0) return GM_OK;
  randint_general_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(perm_seeds, elements, steps,
                                                                                      m_minus_1, n, out);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize((cudaStream_t)stream));
  return GM_OK;
}

int gm_queue_advance_batch(const uint64_t* elements, const double* weights, const int32_t* z0, const double* b0,
                           int64_t n, int32_t k, int32_t steps, uint64_t global_seed, uint64_t stream_salt,
                           uint32_t* perm, double* t_out, uint32_t* s_out, double* b_out, void* stream) {
  g_msg[0] = 0;
  (void)cudaGetLastError();
  if (k < 1 || k > GM_K_MAX || steps < 0 || n < 0)
    return fail(GM_ERR_INVALID_PARAMETER, "gm_queue_advance_batch: k in [1, %d], steps >= 0, n >= 0", GM_K_MAX);
  if (n == 0 || steps == 0) return GM_OK;
  queue_advance_kernel<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
      elements, weights, z0, b0, n, (u32)k, steps, global_seed, global_seed ^ stream_salt, perm, t_out, s_out, b_out);
  CK(cudaGetLastError());
  return GM_OK;
}

int gm_arith_check(int64_t n, uint64_t seed, unsigned long long* counts, void* stream) {
  g_msg[0] = 0;
  (void)cudaGetLastError();
  cudaStream_t st = (cudaStream_t)stream;
  CK(cudaMemsetAsync(counts, 0, 2 * sizeof(unsigned long long), st));
  if (n > 0) arith_check_kernel<<<(unsigned)(num_sms() * 8), 256, 0, st>>>(n, seed, counts);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(st));
  return GM_OK;
}

int gm_log_batch(const double* x, int64_t n, double* out, void* stream) {
  g_msg[0] = 0;
  (void)cudaGetLastError();
  if (n <= 0) return GM_OK;
  log_batch_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(x, n, out);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize((cudaStream_t)stream));
  return GM_OK;
}

int gm_probe_arrival_rate(int64_t n_threads, int32_t iters, int32_t k, double* sink, void* stream) {
  // n_threads threads, each walking C element queues for `iters` arrivals;
  // iters | variant << 24 selects (C, resident CTAs per SM):
  // 0, 2: (2, any)  1: (1, any)  4: (4, any)  5: (1, 8)  6: (2, 6)  7: (1, 6)
  g_msg[0] = 0;
  (void)cudaGetLastError();
  const int variant = iters >> 24;
  iters &= 0xFFFFFF;
  if (k < 128 || k > 65536 || iters < 1 || n_threads < NT || variant == 3 || variant > 7)
    return fail(GM_ERR_INVALID_PARAMETER, "bad probe arguments");
  const unsigned grid = (unsigned)(n_threads / NT);
  cudaStream_t st = (cudaStream_t)stream;
  const u32 kk = (u32)k;
  switch (variant) {
    case 1: arrival_probe_kernel<1><<<grid, NT, 0, st>>>(iters, kk, 0x1234ull, 0x5678ull, sink); break;
    case 4: arrival_probe_kernel<4><<<grid, NT, 0, st>>>(iters, kk, 0x1234ull, 0x5678ull, sink); break;
    case 5: arrival_probe_kernel<1, 8><<<grid, NT, 0, st>>>(iters, kk, 0x1234ull, 0x5678ull, sink); break;
    case 6: arrival_probe_kernel<2, 6><<<grid, NT, 0, st>>>(iters, kk, 0x1234ull, 0x5678ull, sink); break;
    case 7: arrival_probe_kernel<1, 6><<<grid, NT, 0, st>>>(iters, kk, 0x1234ull, 0x5678ull, sink); break;
    default: arrival_probe_kernel<2><<<grid, NT, 0, st>>>(iters, kk, 0x1234ull, 0x5678ull, sink); break;
  }
  CK(cudaGetLastError());
  return GM_OK;
}

int gm_count_arrivals_csr(const void* ids, int id_bits, const void* w, int w_bits,
                          const int64_t* offsets, int64_t n_vec, int32_t k, uint64_t global_seed,
                          const double* tau, unsigned long long* counts, void* stream) {
  g_msg[0] = 0;
  (void)cudaGetLastError();
  int rc = check_common(id_bits, w_bits, k);
  if (rc) return rc;
  if (n_vec <= 0) return GM_OK;
  cudaStream_t st = (cudaStream_t)stream;
  CK(cudaMemsetAsync(counts, 0, (size_t)n_vec * 8, st));
  const unsigned g = (unsigned)n_vec;
  if (id_bits == 32 && w_bits == 32)
    count_le_kernel<u32, float><<<g, NT, 0, st>>>((const u32*)ids, (const float*)w, offsets, n_vec, (u32)k, global_seed, tau, counts);
  else if (id_bits == 32)
    count_le_kernel<u32, double><<<g, NT, 0, st>>>((const u32*)ids, (const double*)w, offsets, n_vec, (u32)k, global_seed, tau, counts);
  else if (w_bits == 32)
    count_le_kernel<u64, float><<<g, NT, 0, st>>>((const u64*)ids, (const float*)w, offsets, n_vec, (u32)k, global_seed, tau, counts);
  else
    count_le_kernel<u64, double><<<g, NT, 0, st>>>((const u64*)ids, (const double*)w, offsets, n_vec, (u32)k, global_seed, tau, counts);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(st));
  return GM_OK;
}

}  // extern "C"
