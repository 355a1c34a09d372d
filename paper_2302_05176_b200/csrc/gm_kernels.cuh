// gm_kernels.cuh -- the FastGM kernels (sm_100a).
//
//   K1 csr4_kernel         batch of CSR vectors (gm_csr4.cuh; configs 1-3,
//                          replaces sketch_fast_counted, sketch.py:218-311).
//   K2 elem_light_kernel + elem_heavy_kernel
//                          one huge element set (a huge vector or an
//                          (id, weight) stream), grid-stride, registers in
//                          global memory (configs 4-5; replaces
//                          sketch_stream / stream_update, stream.py:58-153).
//   K4 merge_kernel        per-register min over sketches, earlier sketch
//                          wins ties (estimate.py:103-125).
//   estimator kernels      register-match counts (estimate.py:47-55).
#pragma once

#include "gm_walk.cuh"

namespace gmk {

constexpr int NT = 256;           // threads per CTA
constexpr int NWARP = NT / 32;

// device-side error word: code in the low 32 bits (gm error enum), the
// first offending vector/element index in the high 32 bits
__device__ __forceinline__ void raise_error(unsigned long long* err, u32 code, u64 where) {
  atomicCAS(err, 0ull, ((unsigned long long)(where & 0xFFFFFFFFull) << 32) | code);
}

template <class T>
__device__ __forceinline__ double load_w(const T* w, int64_t i) {
  return (double)__ldg(&w[i]);
}
template <class T>
__device__ __forceinline__ u64 load_id(const T* ids, int64_t i) {
  return (u64)__ldg(&ids[i]);
}

__device__ __forceinline__ bool weight_ok(double w) {
  // WeightedVector / stream_update validation (sketch.py:57-64, stream.py:63-66)
  return isfinite(w) && w > 0.0 && w >= 1e-300;
}

// Cheap exact pre-filter of an element's first arrival: t1 = -log(u1)/(w k)
// exceeds tau when u1 < exp(-tau w k).  The threshold is taken in fp32 with
// a 2**-12 relative margin (the rounded product and __expf are within ~2**-19 of
// exp(-tau w k) for arguments below 87; beyond that __expf underflows to 0 and
// nothing is skipped), so an element is skipped only if its exact fp64
// arrival is beyond tau: no log, no divide, no permutation for it.
__device__ __forceinline__ bool first_arrival_beyond(u64 ubase, double w, double tau, u32 k) {
  const float x = (float)(tau * w * (double)k);  // fp64 product: no fp32 under/overflow of w or tau
  const double thr = (double)__expf(-x) * (1.0 - 0x1p-12);
  const double u1 = u_open(mix64(ubase + K_STEP));
  return u1 < thr;
}

// threshold for pass `attempt` given total weight W (tau
// bounds the final max register with probability 1 - e^-c)
__device__ __forceinline__ double pass_tau(double W, u32 k, int attempt) {
  const double c = attempt == 0 ? 2.5 : attempt == 1 ? 6.0 : attempt == 2 ? 14.0 : -1.0;
  if (c < 0.0) return __longlong_as_double(0x7FF0000000000000ll);  // +inf: full queues
  return (log((double)k) + c) / W;
}

// ---- K2: one huge element set, registers in global memory ---------------
// light pass: grid-stride, one thread per element; heavy/overflowing
// elements are appended to heavy_list and walked by elem_heavy_kernel.
template <class IdT, class WT, class W = u32>
__global__ void __launch_bounds__(NT)
    elem_light_kernel(const IdT* __restrict__ ids, const WT* __restrict__ wts, int64_t n, u32 k,
                      u64 useed, u64 pseed, const double* __restrict__ tau_p, Reg* regs,
                      int* unset_ctr, u64* __restrict__ heavy_list, int64_t heavy_cap,
                      unsigned long long* heavy_count, unsigned long long* emitted_total,
                      unsigned long long* __restrict__ err) {
  __shared__ W maps[16 * NT];
  const double tau = *tau_p;
  const double light_w = 8.0 / ((double)k * tau);
  u32 emitted = 0;
  W* mymap = maps + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * NT;
  // four coalesced loads in flight per thread, then the cheap first-arrival
  // filter; the rare survivors walk their queues
  for (int64_t i0 = (int64_t)blockIdx.x * NT + threadIdx.x; i0 < n; i0 += 4 * stride) {
    double wv[4];
    u64 idv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = i0 + u * stride;
      wv[u] = i < n ? load_w(wts, i) : 1.0;
      idv[u] = i < n ? load_id(ids, i) : 0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = i0 + u * stride;
      if (i >= n) break;
      const double w = wv[u];
      if (!weight_ok(w)) {
        raise_error(err, 2u, (u64)i);
        continue;
      }
      const u64 id = idv[u];
      if (first_arrival_beyond(useed + id * K_ELEM, w, tau, k)) {
        emitted += 1;
        continue;
      }
      bool ok = false;
      if (w < light_w)
        ok = walk_light<false, W>(id, w, tau, k, useed, pseed, mymap, NT, 16, regs, unset_ctr, emitted);
      if (!ok) {
        const unsigned long long h = atomicAdd(heavy_count, 1ull);
        if ((int64_t)h < heavy_cap) heavy_list[h] = (u64)i;
      }
    }
  }
  if (emitted_total) {
    unsigned long long e = emitted;
#pragma unroll
    for (int o = 16; o; o >>= 1) e += __shfl_xor_sync(0xFFFFFFFFu, e, o);
    if ((threadIdx.x & 31) == 0 && e) atomicAdd(emitted_total, e);
  }
}

// ---- K2 filter pass: stream the element arrays once at HBM speed --------
// Every element's first arrival is tested against the LIST bound tau_hi
// (>= the pass threshold tau) with an fp32 test that needs no
// log, no divide, no MUFU and no fp64: with h23 the top 23 bits of the
// uniform hash, u1 = (h >> 11) 2^-53 + 2^-54 <= (h23 + 1) 2^-23, and
// e^-x >= 1 - x, so the element is skipped when
//   (h23 + 1) < A (1 - x),  A = 2^23 (1 - 2^-16),  x = tau_hi k w,
// evaluated as  float(2^23 + h23) < fma(x, -A, A + 2^23 - 1)  (the left side
// is the bit pattern 0x4B000000 | h23, exact).  Error budget: x carries
// <= 1.2e-7 relative error (two fp32 roundings), the fma rounds by <= 0.5
// (the result is below 2^24, ulp <= 1), so a skip implies
// (h23 + 1) 2^-23 < (1 - 2^-16)(1 - x) + 1.2e-7 x + 2^-24 <= (1 - 2^-17) e^-x
// (for x <= 1/2, 2^-17 (1 - x) >= 3.8e-6 exceeds 1.2e-7 x + 2^-24; beyond,
// e^-x - 1 + x >= 0.1 absorbs them): the element's exact first arrival exceeds
// tau_hi by -log(1 - 2^-17) / (w k) ~ 7.6e-6 / (w k), far beyond fp64
// rounding, so it is skipped only if its exact fp64 first arrival exceeds
// tau_hi.  The margin
// keeps a fraction 2^-16 of the elements whatever their arrival.  For x
// beyond ~1 the right side drops below 2^23 and the element is kept (the
// exact walk decides).  mix64's final xor-shift leaves bits 41..63 unchanged,
// so the last shift is not computed.  Survivors (~k (ln k + c) tau_hi / tau
// per pass) are compacted into a list, so the walk kernel can re-walk the
// list for any tau <= tau_hi (a failed pass) without streaming the element
// arrays again.
__device__ __forceinline__ u32 mix64_hi23(u64 x) {
  x = (x ^ (x >> 30)) * M1;
  x = x ^ (x >> 27);
  return (u32)((x * M2) >> 41);
}

constexpr float FILTER_A = 8388608.0f * (1.0f - 0x1p-16f);           // 2^23 (1 - 2^-16) = 2^23 - 2^7
constexpr float FILTER_B = 8388608.0f * (1.0f - 0x1p-16f) + 8388607.0f;  // A + 2^23 - 1 (exact, < 2^24)

__device__ __forceinline__ bool filter_skip_f(u64 key, float x) {  // key = useed + id K_ELEM + K_STEP
  return __uint_as_float(0x4B000000u | mix64_hi23(key)) < __fmaf_rn(x, -FILTER_A, FILTER_B);
}

// positive, finite (fp32: any such value is >= 1e-300): one integer compare
__device__ __forceinline__ bool weight_ok_f32(float w) { return __float_as_uint(w) - 1u < 0x7F7FFFFFu; }

template <class WT>
__device__ __forceinline__ bool weight_ok_t(WT w) {
  if (sizeof(WT) == 4) {
    const float f = (float)w;
    return f > 0.0f && f < __int_as_float(0x7F800000);  // any positive finite float is >= 1e-300
  }
  return weight_ok((double)w);
}

template <class WT>
__device__ __forceinline__ float filter_x(WT w, float tkf, double tk) {
  return sizeof(WT) == 4 ? tkf * (float)w : (float)(tk * (double)w);
}

// Survivor ids already listed by this CTA in this pass: a repeated id (a
// stream duplicate: same weight, hence the same arrivals) is a register
// no-op, so it is listed once per CTA instead of once per occurrence (Zipf
// streams repeat their hot keys millions of times).  The streaming loop
// drops a kept element whose id sits in its home slot with one shared load
// (a hot key already listed: no call, no atomic); first sightings insert
// (open addressing, 8 probes, then the id is simply listed again).
#ifndef GM_SURV_BITS
#define GM_SURV_BITS 10
#endif
constexpr int SURV_CACHE = 1 << GM_SURV_BITS;

__device__ __forceinline__ u32 surv_slot(u64 id) {
  return (((u32)(id >> 32) * 0x9E3779B1u) ^ ((u32)id * 0x85EBCA6Bu)) >> (32 - GM_SURV_BITS);
}

__device__ __forceinline__ bool surv_cache_first(unsigned long long* cache, u32 h, u64 id) {
  for (int p = 0; p < 8; ++p) {
    const unsigned long long prev = atomicCAS(&cache[h], ~0ull, (unsigned long long)id);
    if (prev == ~0ull) return true;   // inserted: first occurrence here
    if (prev == (unsigned long long)id) return false;
    h = (h + 1) & (SURV_CACHE - 1);
  }
  return true;
}

// A listed survivor: its id and weight (widened to fp64 exactly), so the
// walk kernels read 16 contiguous bytes per entry instead of gathering from
// the element arrays.
struct __align__(16) Surv {
  u64 id;
  double w;
};

// Kept elements are staged per warp in shared memory (WBUF entries) and
// listed in bulk: the streaming loop only stores each kept (id, weight)
// (one warp-wide prefix sum per iteration that keeps anything), and
// flush_kept handles 32 staged entries per step lane-parallel -- insert the
// id into the CTA's id set (first sightings only), one atomic per step for
// the list position.  Per-element work at the moment an element is kept would
// run at 1/32 of the warp's width (lanes hold kept elements one at a time).
#ifndef GM_WBUF
#define GM_WBUF 64
#endif
constexpr int WBUF = GM_WBUF;  // per warp; the filter runs ~4% faster on config 4 with 64 than with 256 entries
static_assert(WBUF >= 32 && WBUF % 8 == 0, "staging area: at least one element per lane, whole lane groups");

__device__ __noinline__ void flush_kept(const Surv* wbuf, u32 wcount, Surv* list, int64_t cap,
                                        unsigned long long* count, unsigned long long* cache) {
  const int lane = threadIdx.x & 31;
  __syncwarp();
  for (u32 j0 = 0; j0 < wcount; j0 += 32) {
    const u32 j = j0 + lane;
    bool kp = j < wcount;
    Surv v{0, 0.0};
    if (kp) {
      v = wbuf[j];
      kp = surv_cache_first(cache, surv_slot(v.id), v.id);
    }
    const unsigned m = __ballot_sync(0xFFFFFFFFu, kp);
    if (!m) continue;
    unsigned long long base = 0;
    if (lane == __ffs(m) - 1) base = atomicAdd(count, (unsigned long long)__popc(m));
    base = __shfl_sync(0xFFFFFFFFu, base, __ffs(m) - 1);
    const unsigned long long pos = base + __popc(m & ((1u << lane) - 1u));
    if (kp && (int64_t)pos < cap) list[pos] = v;
  }
  __syncwarp();
}

// a[e] for a register array and a run-time e, as a select tree (indexing a
// register array with a run-time index would put it in local memory)
template <int NE, class T>
__device__ __forceinline__ T pick(const T (&a)[NE], int e) {
  if constexpr (NE == 1) {
    return a[0];
  } else {
    static_assert(NE == 8, "pick: 1 or 8 entries");
    const T l0 = (e & 1) ? a[1] : a[0], l1 = (e & 1) ? a[3] : a[2];
    const T l2 = (e & 1) ? a[5] : a[4], l3 = (e & 1) ? a[7] : a[6];
    const T m0 = (e & 2) ? l1 : l0, m1 = (e & 2) ? l3 : l2;
    return (e & 4) ? m1 : m0;
  }
}

// stage the kept elements of one iteration (bit e of keep: idv[e], wv[e]);
// returns the warp's new staged count.  Lanes loop over their set bits only
// (a lane keeps one or two of its eight elements at a time).
template <int NE, class WV>
__device__ __forceinline__ u32 stage_kept(u32 keep, const u64 (&idv)[NE], const WV (&wv)[NE], Surv* wbuf,
                                          u32 wcount, Surv* list, int64_t cap, unsigned long long* count,
                                          unsigned long long* cache) {
  const int lane = threadIdx.x & 31;
  const u32 c = __popc(keep);
  u32 incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const u32 v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= o) incl += v;
  }
  const u32 total = __shfl_sync(0xFFFFFFFFu, incl, 31);
  if (wcount + total > (u32)WBUF) {
    flush_kept(wbuf, wcount, list, cap, count, cache);
    wcount = 0;
  }
  if (32 * NE > WBUF && total > (u32)WBUF) {
    // more kept elements in one iteration than the staging area holds (a
    // stream in which nearly everything is kept): stage and flush the lanes
    // in groups of WBUF / NE, each group at most WBUF elements
    constexpr int G = WBUF / NE;
    for (int g = 0; g < 32; g += G) {
      const u32 base = __shfl_sync(0xFFFFFFFFu, incl - c, g);
      const u32 cnt = __shfl_sync(0xFFFFFFFFu, incl, g + G - 1 < 31 ? g + G - 1 : 31) - base;
      if (lane >= g && lane < g + G) {
        u32 p2 = incl - c - base;
        for (u32 m = keep; m; m &= m - 1, ++p2) {
          const int e = __ffs(m) - 1;
          wbuf[p2] = Surv{pick(idv, e), (double)pick(wv, e)};
        }
      }
      flush_kept(wbuf, cnt, list, cap, count, cache);
    }
    return 0;
  }
  u32 pos = wcount + incl - c;
  for (u32 m = keep; m; m &= m - 1, ++pos) {
    const int e = __ffs(m) - 1;
    wbuf[pos] = Surv{pick(idv, e), (double)pick(wv, e)};
  }
  return wcount + total;
}

// resident CTAs per SM the filter's register budget is sized for: 5 with
// 32-bit ids and fp32 weights (48 registers and a 24-byte spill; config 5
// 1.317 -> 1.300 ms), 4 otherwise (64-bit ids need 64 registers: 5 CTAs spill and run
// config 4 8% slower, 3 CTAs 12%)
template <class IdT, class WT>
constexpr int filter_minb() { return sizeof(IdT) == 4 && sizeof(WT) == 4 ? 5 : 4; }
template <class IdT, class WT>
__global__ void __launch_bounds__(NT, filter_minb<IdT, WT>())
    elem_filter_kernel(const IdT* __restrict__ ids, const WT* __restrict__ wts, int64_t n, u32 k, u64 useed,
                       const double* __restrict__ tau_hi_p, Surv* __restrict__ list, int64_t cap,
                       unsigned long long* count, unsigned long long* emitted_total, unsigned long long* err) {
  __shared__ unsigned long long cache[SURV_CACHE];
  __shared__ Surv wbuf_all[NWARP * WBUF];
  for (int i = threadIdx.x; i < SURV_CACHE; i += NT) cache[i] = ~0ull;
  __syncthreads();
  Surv* wbuf = wbuf_all + (threadIdx.x >> 5) * WBUF;
  u32 wcount = 0;
  const double tk = *tau_hi_p * (double)k;
  const float tkf = (float)tk;
  const u64 c0 = useed + K_STEP;
  u32 skipped = 0;
  constexpr bool kVec = sizeof(WT) == 4;  // fp32 weights: float4; ids uint4 (u32) or 2 x ulonglong2 (u64)
  const int64_t tid = (int64_t)blockIdx.x * NT + threadIdx.x, nthr = (int64_t)gridDim.x * NT;
  const bool vec = kVec && (((uintptr_t)ids | (uintptr_t)wts) & 15) == 0;
  int64_t first = 0;
  if (vec) {
    const int64_t nq = n >> 2;  // quads
    const float4* wq = reinterpret_cast<const float4*>(wts);
    // full rounds: every thread has two quads (warp-uniform trip count)
    const int64_t rounds = nq / (2 * nthr);
    for (int64_t r = 0; r < rounds; ++r) {
      const int64_t q0 = r * 2 * nthr + tid, q1 = q0 + nthr;
      u64 idv[8];
      if (sizeof(IdT) == 4) {
        const uint4* iq = reinterpret_cast<const uint4*>(ids);
        const uint4 i0 = __ldcs(&iq[q0]), i1 = __ldcs(&iq[q1]);
        idv[0] = i0.x; idv[1] = i0.y; idv[2] = i0.z; idv[3] = i0.w;
        idv[4] = i1.x; idv[5] = i1.y; idv[6] = i1.z; idv[7] = i1.w;
      } else {
        const ulonglong2* iq = reinterpret_cast<const ulonglong2*>(ids);
        const ulonglong2 a0 = __ldcs(&iq[2 * q0]), a1 = __ldcs(&iq[2 * q0 + 1]);
        const ulonglong2 b0 = __ldcs(&iq[2 * q1]), b1 = __ldcs(&iq[2 * q1 + 1]);
        idv[0] = a0.x; idv[1] = a0.y; idv[2] = a1.x; idv[3] = a1.y;
        idv[4] = b0.x; idv[5] = b0.y; idv[6] = b1.x; idv[7] = b1.y;
      }
      const float4 w0 = __ldcs(&wq[q0]), w1 = __ldcs(&wq[q1]);
      const float wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
      u32 keep, bad = 0;
      if constexpr (sizeof(IdT) == 4) {
        // skip = the test passes and w > 0: a zero, negative, infinite or NaN
        // weight is never skipped (the fma gives -inf or NaN for the last two),
        // so weights are validated on the kept elements only.  (With u64 ids
        // the extra live values of that path spill at the 64-register budget:
        // there every weight is validated up front.)
        u32 skm = 0;
#pragma unroll
        for (int e = 0; e < 8; ++e)
          skm |= (u32)(filter_skip_f(c0 + idv[e] * K_ELEM, tkf * wv[e]) & (wv[e] > 0.0f)) << e;
        keep = ~skm & 0xFFu;
        skipped += __popc(skm);
      } else {
        u32 okm = 0, skm = 0;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          okm |= (u32)weight_ok_f32(wv[e]) << e;
          skm |= (u32)filter_skip_f(c0 + idv[e] * K_ELEM, tkf * wv[e]) << e;
        }
        keep = okm & ~skm;
        bad = ~okm & 0xFFu;
        skipped += __popc(okm & skm);
      }
      if (keep) {  // (validate;) drop ids this CTA has listed already (hot stream keys): set bits only
        const volatile unsigned long long* vc = cache;
        for (u32 m = keep; m; m &= m - 1) {
          const int e = __ffs(m) - 1;
          const u64 id = pick(idv, e);
          if (sizeof(IdT) == 4 && !weight_ok_f32(pick(wv, e))) {
            bad |= 1u << e;
            keep &= ~(1u << e);
          } else if (vc[surv_slot(id)] == (unsigned long long)id) {
            keep &= ~(1u << e);
          }
        }
      }
      // bit e: quad q0 (e < 4) or q1 (e >= 4), element e & 3
      if (__any_sync(0xFFFFFFFFu, keep != 0u))
        wcount = stage_kept(keep, idv, wv, wbuf, wcount, list, cap, count, cache);
      if (bad) raise_error(err, 2u, (u64)((__ffs(bad) - 1 < 4 ? 4 * q0 : 4 * q1 - 4) + __ffs(bad) - 1));
    }
    first = rounds * 2 * nthr * 4;
  }
  // scalar path: everything (no vector loads) or what the full rounds left
  for (int64_t i0 = first + tid; i0 - tid < n; i0 += nthr) {
    u32 keep = 0, bad = 0;
    u64 idv[1] = {0};
    WT wv[1] = {WT(1)};
    if (i0 < n) {
      wv[0] = __ldcs(&wts[i0]);
      idv[0] = (u64)__ldcs(&ids[i0]);
      const bool ok = weight_ok_t(wv[0]);
      const bool sk = ok && filter_skip_f(c0 + idv[0] * K_ELEM, filter_x(wv[0], tkf, tk));
      bad = !ok;
      keep = ok && !sk;
      skipped += sk;
    }
    if (__any_sync(0xFFFFFFFFu, keep != 0u)) wcount = stage_kept(keep, idv, wv, wbuf, wcount, list, cap, count, cache);
    if (bad) raise_error(err, 2u, (u64)i0);
  }
  if (wcount) flush_kept(wbuf, wcount, list, cap, count, cache);
  if (emitted_total) {
    unsigned long long e = skipped;
#pragma unroll
    for (int o = 16; o; o >>= 1) e += __shfl_xor_sync(0xFFFFFFFFu, e, o);
    if ((threadIdx.x & 31) == 0 && e) atomicAdd(emitted_total, e);
  }
}

// survivors of the filter: walk light elements lane-parallel (as the fused
// light kernel does); heavy or table-full ones go to the heavy list (as
// list positions).  A listed element whose first arrival lies beyond this
// pass's tau (the list was built for tau_hi >= tau) emits that one arrival
// and stops.
template <class W = u32>
__global__ void __launch_bounds__(NT)
    elem_survivor_kernel(const Surv* __restrict__ list, const unsigned long long* count, int64_t cap, u32 k,
                         u64 useed, u64 pseed, const double* __restrict__ tau_p, Reg* regs, int* unset_ctr,
                         u64* __restrict__ heavy_list, int64_t heavy_cap, unsigned long long* heavy_count,
                         unsigned long long* emitted_total) {
  __shared__ W maps[16 * NT];
  const double tau = *tau_p;
  const double light_w = 8.0 / ((double)k * tau);
  const int64_t m = min((int64_t)*count, cap);
  u32 emitted = 0;
  W* mymap = maps + threadIdx.x;
  for (int64_t j = (int64_t)blockIdx.x * NT + threadIdx.x; j < m; j += (int64_t)gridDim.x * NT) {
    const Surv v = list[j];
    // the list was built for tau_hi >= tau: the filter's fp32 test against this
    // pass's tau drops most entries beyond it without the exact arithmetic
    if (filter_skip_f(useed + K_STEP + v.id * K_ELEM, (float)(tau * (double)k * v.w)) & (v.w > 0.0)) {
      emitted += 1;
      continue;
    }
    bool ok = false;
    if (v.w < light_w) ok = walk_light<false, W>(v.id, v.w, tau, k, useed, pseed, mymap, NT, 16, regs, unset_ctr, emitted);
    if (!ok) {
      const unsigned long long h = atomicAdd(heavy_count, 1ull);
      if ((int64_t)h < heavy_cap) heavy_list[h] = (u64)j;
    }
  }
  if (emitted_total) {
    unsigned long long e = emitted;
#pragma unroll
    for (int o = 16; o; o >>= 1) e += __shfl_xor_sync(0xFFFFFFFFu, e, o);
    if ((threadIdx.x & 31) == 0 && e) atomicAdd(emitted_total, e);
  }
}

// one warp per heavy element; dense arrays in global scratch, one per warp;
// the last CTA stores the registers to (y_out, s_out).
// Heavy-list entries index the survivor list when `surv` is given (after the
// filter), the element arrays otherwise (after the fused light kernel).
template <class IdT, class WT, class W = u32>
__global__ void __launch_bounds__(NT)
    elem_heavy_kernel(const IdT* __restrict__ ids, const WT* __restrict__ wts, const Surv* __restrict__ surv,
                      u32 k, u64 useed, u64 pseed, const double* __restrict__ tau_p, Reg* regs, int* unset_ctr,
                      const u64* __restrict__ heavy_list, const unsigned long long* heavy_count,
                      int64_t heavy_cap, W* __restrict__ dense_global,
                      unsigned long long* emitted_total, unsigned* done, double* y_out, u64* s_out) {
  __shared__ double scan_all[NWARP * 32];
  __shared__ int prov_all[NWARP * 32];
  const double tau = *tau_p;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nh = min((int64_t)*heavy_count, heavy_cap);
  const int64_t gw = (int64_t)blockIdx.x * NWARP + warp;
  W* dense = dense_global + (size_t)gw * k;
  u32 stamp = 0, emitted = 0;
  for (int64_t h = gw; h < nh; h += (int64_t)gridDim.x * NWARP) {
    const int64_t i = (int64_t)heavy_list[h];
    if (++stamp == (FyWord<W>::BIG ? 0xFFFFFFFFu : 0x10000u)) {
      for (u32 q = lane; q < k; q += 32) dense[q] = 0;
      __syncwarp();
      stamp = 1;
    }
    u32 em = 0;
    // heavy-list entries are survivor-list positions (surv != null) or element indices
    const u64 id = surv ? surv[i].id : load_id(ids, i);
    const double w = surv ? surv[i].w : load_w(wts, i);
    walk_warp<false>(id, w, tau, k, useed, pseed, dense, stamp,
                     scan_all + warp * 32, prov_all + warp * 32, regs, unset_ctr, em, 0u, 0.0, nullptr, 0u,
                     &gm_glog_tab[0][0]);
    if (lane == 0) emitted += em;
  }
  // leave the scratch clean for the next launch
  __syncwarp();
  if (stamp)
    for (u32 q = lane; q < k; q += 32) dense[q] = 0;
  if (emitted_total && lane == 0 && emitted) atomicAdd(emitted_total, (unsigned long long)emitted);
  // the last CTA to finish writes the registers out (y, s): no separate
  // store launch; `done` is left at 0 for the next launch
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  const ulonglong2* rv = reinterpret_cast<const ulonglong2*>(regs);
  for (u32 j0 = threadIdx.x; j0 < k; j0 += 8 * NT) {  // L2 reads (the CAS results live there), 8 in flight
    ulonglong2 r[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (j0 + u * NT < k) r[u] = __ldcg(rv + j0 + u * NT);
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (j0 + u * NT < k) {
        y_out[j0 + u * NT] = __longlong_as_double((long long)r[u].x);
        s_out[j0 + u * NT] = r[u].y;
      }
  }
  if (threadIdx.x == 0) *done = 0u;
}

__global__ void init_regs_kernel(Reg* regs, u32 k, int* unset_ctr) {
  for (u32 j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x) {
    regs[j].y = INF_BITS;
    regs[j].id = NO_ID;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *unset_ctr = (int)k;
}

// registers from caller-provided (y, s) (accumulate mode); counts unset ones
__global__ void load_regs_kernel(Reg* regs, u32 k, const double* y, const u64* s, int* unset_ctr) {
  for (u32 j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x) {
    const u64 yb = (u64)__double_as_longlong(y[j]);
    regs[j].y = yb;
    regs[j].id = s[j];
    if (yb == INF_BITS) atomicAdd(unset_ctr, 1);
  }
}

// GM_FLAG_ACCUMULATE: after a pass at tau, the registers that are not yet
// final -- unset, or above tau (an arrival of the new elements in (tau, y_j)
// could still lower y_j; registers loaded from an earlier sketch are set but
// not bounded by this pass's tau).  Overwrites the counter the walkers
// decrement; one block.
__global__ void __launch_bounds__(1024) count_unfinished_kernel(const Reg* regs, u32 k, const double* tau_p,
                                                                int* out) {
  const double tau = *tau_p;
  int c = 0;
  for (u32 j = threadIdx.x; j < k; j += blockDim.x) {
    const u64 y = __ldcg(&regs[j].y);
    c += (y == INF_BITS || __longlong_as_double((long long)y) > tau) ? 1 : 0;
  }
  c = __reduce_add_sync(0xFFFFFFFFu, c);
  __shared__ int part[32];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += part[i];
    *out = t;
  }
}

__global__ void store_regs_kernel(const Reg* regs, u32 k, double* y, u64* s) {
  for (u32 j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x) {
    y[j] = __longlong_as_double((long long)regs[j].y);
    s[j] = regs[j].id;
  }
}

// First pass threshold and list bound from the sampled weights (per-block
// partials: all sampled weight, and the sampled weight of ids seen for the
// first time in the sample; both scaled by n / sampled items).  tau = (ln k + 3) / W
// with W the duplicate-corrected estimate; the filter lists every element
// whose first arrival is <= tau_hi = R tau, R = 2 x the sample's duplication
// ratio (in [2, 256]): a stream whose sample under-counts its duplicates (a
// Zipf stream: the sample sees few repeats of the rare keys) gets a first
// tau that is too small, and the next pass re-walks the list with a larger
// tau instead of streaming the input again (gm_capi.cu run_elements).
// (one block of 256 threads; the partials are summed in a fixed order)
struct TauArgs {
  double* tau;              // out: [0] tau, [1] W sampled, [2] W distinct, [3] tau_hi
  const double* part;       // per-block partials of the sample
  int nblocks;
  u32 k;
  double scale;             // n / sampled items
  double tau_scale, r_fixed;  // test knobs (1, 0 by default)
  unsigned long long* ctr4;   // cleared: heavy count, emitted, list count, spare
  int walk_hi;                // walk the list at tau_hi whatever the duplication (one-pass calls)
};

// (one block of 256 threads; the partials are summed in a fixed order)
__device__ __forceinline__ void tau_block(const TauArgs& A) {
  double* tau = A.tau;
  const u32 k = A.k;
  __shared__ double red[2][256];
  if (threadIdx.x < 4) A.ctr4[threadIdx.x] = 0ull;
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < A.nblocks; i += 256) {
    a += __ldcg(A.part + 2 * i);
    b += __ldcg(A.part + 2 * i + 1);
  }
  red[0][threadIdx.x] = a;
  red[1][threadIdx.x] = b;
  __syncthreads();
  for (int h = 128; h; h >>= 1) {
    if ((int)threadIdx.x < h) {
      red[0][threadIdx.x] += red[0][threadIdx.x + h];
      red[1][threadIdx.x] += red[1][threadIdx.x + h];
    }
    __syncthreads();
  }
  if (threadIdx.x) return;
  const double lk = log((double)k);
  double all = red[0][0], dist = red[1][0];
  all *= A.scale;
  dist *= A.scale;
  tau[1] = all;
  tau[2] = dist;
  const double W = dist > 0.0 ? dist : all;
  const double ratio = (dist > 0.0 && all > dist) ? all / dist : 1.0;
  const double R = A.r_fixed > 0.0 ? A.r_fixed : fmin(fmax(2.0 * ratio, 2.0), 256.0);
  const double t0 = A.tau_scale * (lk + 3.0) / W;
  tau[3] = R * t0;
  // a stream with visible duplication walks the list at tau_hi right away:
  // its first tau would come from an over-estimated W, and a failed walk costs
  // a host round trip and a second walk (the list walk is ~1 arrival per
  // listed element either way)
  tau[0] = ((ratio > 1.5 || A.walk_hi) && A.r_fixed <= 0.0) ? tau[3] : t0;
}

// Blocked sample of the stream: block b of the grid reads the contiguous
// items [b n / G, b n / G + L) (L = min(SAMPLE_RUN, n / G), coalesced), and
// sums their weights and the weights of ids not seen before in the sample
// (a global hash set of `tcap` slots, power of two, all ~0 on entry, behind a
// run-local shared-memory set, and used only by runs that repeat an id
// themselves; id ~0 is never inserted and counts as new).  Per-block partials out[2b], out[2b+1];
// the last block sums them, scales by n / sampled and sets tau and tau_hi
// (tau_block).  With `regs` given the kernel also initialises the k
// registers and the unset counter.
constexpr int SAMPLE_RUN = 256;  // <= the launch's 256 threads: one item per thread

template <class IdT, class WT>
__global__ void __launch_bounds__(256) weight_sample_kernel(const IdT* __restrict__ ids, const WT* __restrict__ wts,
                                                            int64_t n, unsigned long long* table, u32 tcap, double* out,
                                                            Reg* regs, u32 k, int* unset_ctr, TauArgs targs,
                                                            unsigned* done) {
  if (regs) {  // fresh registers (one launch fewer)
    const u32 g0 = blockIdx.x * blockDim.x + threadIdx.x;
    for (u32 g = g0; g < k; g += gridDim.x * blockDim.x) {
      regs[g].y = INF_BITS;
      regs[g].id = NO_ID;
    }
    if (g0 == 0) *unset_ctr = (int)k;
  }
  const int64_t lo = (int64_t)blockIdx.x * n / gridDim.x;
  const int64_t hi = min(lo + (int64_t)SAMPLE_RUN, ((int64_t)blockIdx.x + 1) * n / gridDim.x);
  // the run is first deduplicated in a shared-memory set (hot keys repeat
  // within a run), so only the run's distinct ids go to the global set, with
  // one atomic each (a global CAS is the cost of this kernel)
  constexpr u32 LCAP = 2 * SAMPLE_RUN;
  __shared__ unsigned long long lset[LCAP];
  for (u32 i = threadIdx.x; i < LCAP; i += blockDim.x) lset[i] = ~0ull;
  __syncthreads();
  // one item per thread (SAMPLE_RUN <= blockDim.x)
  double s = 0.0, sd = 0.0;
  const int64_t i = lo + threadIdx.x;
  bool fresh = false;
  u64 id = 0, hh = 0;
  if (i < hi) {
    const double w = (double)wts[i];
    if (isfinite(w) && w > 0.0) {
      s = w;
      fresh = true;
      id = (u64)ids[i];
      if (id != ~0ull && tcap) {
        hh = mix64(id);
        u32 h = (u32)hh & (LCAP - 1);
        for (;;) {  // run-local set (LCAP >= 2 x the run: always has room)
          const unsigned long long prev = atomicCAS(&lset[h], ~0ull, (unsigned long long)id);
          if (prev == ~0ull) break;
          if (prev == (unsigned long long)id) {
            fresh = false;
            break;
          }
          h = (h + 1) & (LCAP - 1);
        }
      }
    }
  }
  // a run without any repeat goes no further (a stream without duplicates
  // then costs no global atomics); a run with repeats checks its distinct ids
  // against the sample-wide set
  const bool run_dups = __syncthreads_or(s > 0.0 && !fresh);
  if (run_dups && fresh && id != ~0ull && tcap) {
    u32 h = (u32)(hh >> 32) & (tcap - 1);
    while (fresh) {  // sample-wide set
      const unsigned long long prev = atomicCAS(&table[h], ~0ull, (unsigned long long)id);
      if (prev == ~0ull) break;
      if (prev == (unsigned long long)id) fresh = false;
      h = (h + 1) & (tcap - 1);
    }
  }
  if (fresh) sd = s;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    s += __shfl_xor_sync(0xFFFFFFFFu, s, o);
    sd += __shfl_xor_sync(0xFFFFFFFFu, sd, o);
  }
  __shared__ double red[2][32];
  const int warp = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    red[0][warp] = s;
    red[1][warp] = sd;
  }
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) {  // per-block partials, summed in block order by the last block (deterministic)
    double a = 0.0, b = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
      a += red[0][i];
      b += red[1][i];
    }
    out[2 * blockIdx.x] = a;
    out[2 * blockIdx.x + 1] = b;
    __threadfence();
    last = atomicAdd(done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  tau_block(targs);  // the pass threshold and the list bound (one launch fewer)
  if (threadIdx.x == 0) *done = 0u;
}

__global__ void merge_kernel(const double* __restrict__ y_in, const u64* __restrict__ s_in,
                             int64_t n_sk, u32 k, double* __restrict__ y_out,
                             u64* __restrict__ s_out) {
  for (u32 j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x) {
    double y = y_in[j];
    u64 s = s_in[j];
    for (int64_t r = 1; r < n_sk; ++r) {
      const double t = y_in[r * k + j];
      if (t < y) {  // strict: earlier sketch wins ties (estimate.py:121-124)
        y = t;
        s = s_in[r * k + j];
      }
    }
    y_out[j] = y;
    s_out[j] = s;
  }
}

// ---- estimators: register matches of sketch pairs (estimate.py:54) ----
__global__ void match_count_kernel(const u64* __restrict__ s_a, const u64* __restrict__ s_b,
                                   int64_t n_pairs, u32 k, int32_t* __restrict__ matches) {
  const int64_t p = blockIdx.x;
  if (p >= n_pairs) return;
  int c = 0;
  for (u32 j = threadIdx.x; j < k; j += blockDim.x) c += s_a[p * k + j] == s_b[p * k + j];
#pragma unroll
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
  __shared__ int part[32];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += part[i];
    matches[p] = t;
  }
}

// ---- estimators: exactly rounded register sums (math.fsum, estimate.py:100)
// One CTA per sketch.  Every y >= 0 is m * 2^e with a 53-bit integer m; it
// is added exactly into a fixed-point superaccumulator of 32-bit digits
// (int64 limbs in shared memory absorb the carries of up to 2^31 adds), the
// carries are propagated once, and the top digits are rounded to nearest
// even with a sticky bit: the correctly rounded sum, i.e. math.fsum's.
// card = (k - 1) / sum (an IEEE divide, like the reference's).  A +inf
// register gives +inf (card 0); a negative or NaN one gives NaN.
constexpr int SUM_DIGITS = 68;  // 32 * 68 bits >= 1074 + 1024 + 53 + carry room

__global__ void __launch_bounds__(256) exact_sum_kernel(const double* __restrict__ y, int64_t n_sk, u32 k,
                                                        double* __restrict__ sum_out,
                                                        double* __restrict__ card_out) {
  __shared__ unsigned long long acc[SUM_DIGITS];
  __shared__ int special;  // bit 0: +inf seen, bit 1: NaN / negative seen
  const int64_t sk = blockIdx.x;
  if (sk >= n_sk) return;
  for (int i = threadIdx.x; i < SUM_DIGITS; i += blockDim.x) acc[i] = 0;
  if (threadIdx.x == 0) special = 0;
  __syncthreads();
  for (u32 j = threadIdx.x; j < k; j += blockDim.x) {
    const double v = y[sk * (int64_t)k + j];
    const u64 b = (u64)__double_as_longlong(v);
    const int ex = (int)((b >> 52) & 0x7FF);
    if ((b >> 63) && v != 0.0) { atomicOr(&special, 2); continue; }
    if (ex == 0x7FF) { atomicOr(&special, (b & 0xFFFFFFFFFFFFFull) ? 2 : 1); continue; }
    const u64 m = (b & 0xFFFFFFFFFFFFFull) | (ex ? (1ull << 52) : 0ull);
    if (!m) continue;
    const int p = ex ? ex - 1 : 0;  // bit position of m's lsb above 2^-1074
    const unsigned __int128 sh = (unsigned __int128)m << (p & 31);
    const int q = p >> 5;
    atomicAdd(&acc[q], (unsigned long long)(u32)sh);
    atomicAdd(&acc[q + 1], (unsigned long long)(u32)(sh >> 32));
    atomicAdd(&acc[q + 2], (unsigned long long)(u32)(sh >> 64));
  }
  __syncthreads();
  if (threadIdx.x) return;
  double total;
  if (special & 2) {
    total = __longlong_as_double(0x7FF8000000000000ll);
  } else if (special & 1) {
    total = __longlong_as_double(0x7FF0000000000000ll);
  } else {
    unsigned long long carry = 0;
    int top = -1;
    for (int i = 0; i < SUM_DIGITS; ++i) {
      const unsigned long long t = acc[i] + carry;
      acc[i] = t & 0xFFFFFFFFull;
      carry = t >> 32;
      if (acc[i]) top = i;
    }
    if (top < 0) {
      total = 0.0;
    } else {
      // the top three digits as a 96-bit integer, the rest as a sticky bit
      unsigned __int128 mant = 0;
      bool sticky = false;
      const int lo = top >= 2 ? top - 2 : 0;
      for (int i = top; i >= lo; --i) mant = (mant << 32) | acc[i];
      for (int i = lo - 1; i >= 0; --i) sticky |= acc[i] != 0;
      const int msb = 127 - (mant >> 64 ? __clzll((long long)(u64)(mant >> 64)) : 64 + __clzll((long long)(u64)mant));
      int e = 32 * lo - 1074;  // weight of mant's lsb
      u64 r;
      if (msb > 52) {
        const int shift = msb - 52;
        r = (u64)(mant >> shift);
        const unsigned __int128 rem = mant & (((unsigned __int128)1 << shift) - 1);
        const unsigned __int128 half = (unsigned __int128)1 << (shift - 1);
        if (rem > half || (rem == half && (sticky || (r & 1)))) ++r;
        e += shift;
        if (r >> 53) { r >>= 1; ++e; }
      } else {
        r = (u64)mant;  // exact: fewer than 54 significant bits and no lower digits
      }
      total = scalbn((double)r, e);  // exact for the normal sums registers produce
    }
  }
  sum_out[sk] = total;
  if (card_out) card_out[sk] = __ddiv_rn((double)(k - 1), total);
}

// s narrowed to 32 bits (GM_FLAG_S32 host outputs; an unset register's
// UINT64_MAX becomes 0xFFFFFFFF)
__global__ void narrow_u32_kernel(const u64* __restrict__ in, u32* __restrict__ out, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (u32)in[i];
}

// ---- K0 test kernels: the keyed streams element by element ----
__global__ void uniform_kernel(const u64* seeds, const u64* elems, const u64* steps, int64_t n,
                               double* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = u_open(mix64(seeds[i] + elems[i] * K_ELEM + steps[i] * K_STEP));
}

__global__ void randint_kernel(const u64* pseeds, const u64* elems, const u64* steps,
                               const u32* ks, int64_t n, u32* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = perm_draw(pseeds[i] + elems[i] * K_ELEM, (u32)steps[i], ks[i]);
}

// rand_int_between over any range m <= 2^64 (randgen.py:122-143): offset
// x mod m of the first accepted rehash x of the (element, step) key, with the
// reference's rejection bound 2^64 - (2^64 mod m).  m_minus_1 = m - 1 (so
// m = 2^64 is representable).  Exact 64-bit remainders (the sketch kernels
// draw with m <= 65536 through perm_draw).
__global__ void randint_general_kernel(const u64* pseeds, const u64* elems, const u64* steps,
                                       const u64* m_minus_1, int64_t n, u64* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const u64 key = pseeds[i] + elems[i] * K_ELEM + steps[i] * K_STEP;
  const u64 mm1 = m_minus_1[i];
  u64 x = mix64(key);
  if (mm1 == ~0ull) {  // m = 2^64: every x is accepted, x mod 2^64 = x
    out[i] = x;
    return;
  }
  const u64 m = mm1 + 1;
  const u64 r = (~0ull % m + 1) % m;  // 2^64 mod m
  for (u64 attempt = 1; r != 0 && x > ~0ull - r; ++attempt) x = mix64(key + attempt * K_RETRY);
  out[i] = x % m;
}

// ElementQueueState / next_order_statistic (randgen.py:210-271) on the device:
// queue i emits `steps` order statistics from its cursor (z0[i] emitted, last
// time b0[i]), swapping its dense Fisher-Yates array perm[i*k .. i*k+k)
// (values 1..k) in place: the reference's _run_queue arithmetic
// (randgen.py:181-203) with glibc's log.  One thread per queue.
__global__ void queue_advance_kernel(const u64* __restrict__ elems, const double* __restrict__ w,
                                     const int32_t* __restrict__ z0, const double* __restrict__ b0, int64_t n, u32 k,
                                     int32_t steps, u64 useed, u64 pseed, u32* __restrict__ perm,
                                     double* __restrict__ t_out, u32* __restrict__ s_out, double* __restrict__ b_out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const u64 ubase = useed + elems[i] * K_ELEM, pbase = pseed + elems[i] * K_ELEM;
  u32* P = perm + i * (int64_t)k;
  double b = b0[i];
  for (int32_t q = 0; q < steps; ++q) {
    const u32 z = (u32)z0[i] + (u32)q + 1u;
    const double L = -log_pos(u_open(mix64(ubase + (u64)z * K_STEP)));
    b = __dadd_rn(b, __ddiv_rn(L, __dmul_rn(w[i], (double)(k - z + 1))));
    const u32 jpos = (k > 65536u ? perm_draw_big(pbase, z, k) : perm_draw(pbase, z, k)) - 1;
    const u32 vz = P[z - 1];
    P[z - 1] = P[jpos];
    P[jpos] = vz;
    t_out[i * steps + q] = b;
    s_out[i * steps + q] = P[z - 1];
  }
  b_out[i] = b;
}

// ---- arithmetic self-check: ddiv_fast == __ddiv_rn on the fast range, and
// log_pos within 1 ulp of CUDA's log, over keyed random inputs ----
__global__ void arith_check_kernel(int64_t n, u64 seed, unsigned long long* counts) {
  unsigned long long bad_div = 0, bad_log = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const u64 a = mix64(seed + (u64)i * K_ELEM), b = mix64(a ^ K_STEP), c = mix64(b + K_RETRY);
    const double u = u_open(a);
    const double L = -log_pos(u);
    // divisor: w in [2**-940, 2**900] log-uniform-ish, times an integer m <= 65536
    const int ex = (int)(b % 1840u) - 940;
    const double w = ldexp(1.0 + (double)(c >> 12) * 0x1p-52, ex);
    const double D = __dmul_rn(w, (double)(1u + (u32)(c & 0xFFFFu)));
    const double q1 = ddiv_fast(L, D), q2 = __ddiv_rn(L, D);
    bad_div += __double_as_longlong(q1) != __double_as_longlong(q2) && !(q1 == 0.0 && q2 == 0.0);
    const double l2 = log(u);
    const long long dl = __double_as_longlong(-L) - __double_as_longlong(l2);
    bad_log += (dl > 1 || dl < -1) && !(L == 0.0 && l2 == 0.0);
  }
  for (int o = 16; o; o >>= 1) {
    bad_div += __shfl_xor_sync(0xFFFFFFFFu, bad_div, o);
    bad_log += __shfl_xor_sync(0xFFFFFFFFu, bad_log, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&counts[0], bad_div);
    atomicAdd(&counts[1], bad_log);
  }
}

// device log of given inputs (parity tests compare it with glibc's)
__global__ void log_batch_kernel(const double* x, int64_t n, double* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = log_pos(x[i]);
}

// ---- diagnostics ----
// Speed-of-light probe for the arrival generator (the roofline K1 is
// reported against): every thread walks C independent element queues with
// exactly the lane step's arithmetic per arrival -- the uniform hash,
// u_open, the glibc-clone log with the table in shared memory, the rounded
// product w (k - z + 1), the branch-free divide, the prefix add, and the
// permutation hash with the 64-bit Barrett reduction from a shared-memory
// table -- with no pruning, no Fisher-Yates table, no register update, no
// queue bookkeeping and no memory traffic.  C chains per thread give the
// scheduler independent work (ILP) on top of full occupancy.
template <int C, int MINB = 1>
__global__ void __launch_bounds__(NT, MINB) arrival_probe_kernel(int iters, u32 k, u64 useed, u64 pseed, double* sink) {
  __shared__ __align__(16) double ltab[256];
  __shared__ u64 mtab64[128];
  for (u32 i = threadIdx.x; i < 256; i += NT) ltab[i] = gm_glog_tab[i >> 1][i & 1];
  for (u32 z = threadIdx.x; z < 128; z += NT) mtab64[z] = barrett_magic64(k - z + 1);
  __syncthreads();
  u64 ub[C], pb[C];
  double b[C], w[C];
  u32 acc = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const u64 id = ((u64)blockIdx.x * NT + threadIdx.x) * C + c;
    ub[c] = useed + id * K_ELEM;
    pb[c] = pseed + id * K_ELEM;
    b[c] = 0.0;
    w[c] = 1.0 + (double)((threadIdx.x + c) & 7);
  }
  for (int i = 0; i < iters; ++i) {
    const u32 z = 1u + ((u32)i & 126u);
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const u64 x = mix64(ub[c] + (u64)z * K_STEP);
      const double L = -log_pos_t(u_open(x), ltab);
      const double D = __dmul_rn(w[c], (double)(k - z + 1));
      b[c] = __dadd_rn(b[c], ddiv_fast(L, D));
      const u64 g = mix64(pb[c] + (u64)z * K_STEP);
      acc += z + mod_barrett64(g, k - z + 1, mtab64[z]);
    }
  }
  double t = 0.0;
#pragma unroll
  for (int c = 0; c < C; ++c) t += b[c];
  if (t == -1.0 || acc == 0xFFFFFFFFu) sink[0] = t + (double)acc;
}

// Number of arrivals t <= tau_v of every element of every CSR vector
// (times only; the algorithmic survivor count of a pass at tau_v).
template <class IdT, class WT>
__global__ void __launch_bounds__(NT) count_le_kernel(const IdT* __restrict__ ids,
                                                      const WT* __restrict__ wts,
                                                      const int64_t* __restrict__ offsets,
                                                      int64_t n_vec, u32 k, u64 useed,
                                                      const double* __restrict__ tau,
                                                      unsigned long long* __restrict__ counts) {
  const int64_t v = blockIdx.x;
  if (v >= n_vec) return;
  const double t_v = tau[v];
  unsigned long long c = 0;
  for (int64_t i = offsets[v] + threadIdx.x; i < offsets[v + 1]; i += NT) {
    const u64 ubase = useed + load_id(ids, i) * K_ELEM;
    const double w = load_w(wts, i);
    double b = 0.0;
    for (u32 z = 1; z <= k; ++z) {
      b = __dadd_rn(b, spacing(ubase, z, w, k));
      if (b > t_v) break;
      ++c;
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(&counts[v], c);
}

}  // namespace gmk
