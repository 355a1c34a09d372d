// gm_walk.cuh -- element-queue walkers (the device form of _run_queue,
// randgen.py:158-207, driven to a threshold instead of a fixed cursor).
//
// A walker emits an element's arrivals in ascending order and folds every
// arrival t <= tau into the registers; it stops at the first arrival > tau
// (that arrival and all later ones exceed tau).  When every register is set
// at the end of a pass, tau bounds the final maximum register, so every
// arrival that can win a register was emitted and the sketch equals
// sketch_naive's (the schedule-independence sketch_fast relies on,
// sketch.py:277-282).  Re-emitting an arrival is a no-op on the registers,
// so a pass can be repeated with a larger tau without undoing anything.
//
// The Fisher-Yates state (LazyPermutation, randgen.py:146-155) is sparse:
//  * light walker (one thread per element): a linear list of
//    (position, value) pairs in the thread's shared-memory slice; the entry
//    at position z-1 dies at step z, so the list holds only positions >= z.
//  * warp walker (32 steps of one element per iteration): a stamped dense
//    array of k words; the 32 swaps of a batch are resolved in parallel by
//    provider chains (see walk_warp).
#pragma once

#include <type_traits>
#include <utility>

#include "gm_core.cuh"

namespace gmk {

struct WalkStats {
  u32 emitted;  // arrivals computed (accepted + the terminating one)
};

// ---- light walker -------------------------------------------------------
// map: this thread's slice, entry e at map[e * stride]; entries are
// (pos << 16) | (val - 1).  Returns false if the list overflowed (the caller
// re-walks the element with the warp walker; registers already updated
// stay valid).
template <bool kSharedRegs, class W = u32>
__device__ __forceinline__ bool walk_light(u64 id, double w, double tau, u32 k, u64 useed,
                                           u64 pseed, W* map, int stride, int cap, Reg* regs,
                                           int* unset_ctr, u32& emitted) {
  constexpr int SH = FyWord<W>::SH;
  constexpr W LOW = FyWord<W>::LOW;
  const u64 ubase = useed + id * K_ELEM;
  const u64 pbase = pseed + id * K_ELEM;
  const bool fast = w_fast(w);  // the branch-free divide gives the IEEE quotient in this range
  double b = 0.0;
  int nl = 0;
  u32 z = 0;
  while (z < k) {
    ++z;
    const double t = __dadd_rn(b, fast ? spacing_t<true>(ubase, z, w, k) : spacing_t<false>(ubase, z, w, k));
    if (t > tau) break;
    b = t;
    const u32 j = perm_draw_w<W>(pbase, z, k);
    const u32 zi = z - 1, ji = j - 1;
    u32 vz = zi + 1, vj = ji + 1;
    int sz = -1, sj = -1;
    for (int e = 0; e < nl; ++e) {
      const W ent = map[e * stride];
      const u32 p = (u32)(ent >> SH);
      if (p == zi) {
        vz = (u32)(ent & LOW) + 1;
        sz = e;
      }
      if (p == ji) {
        vj = (u32)(ent & LOW) + 1;
        sj = e;
      }
    }
    // perm[zi] <- vj (dead from now on), perm[ji] <- vz
    if (ji != zi) {
      const W nent = ((W)ji << SH) | (W)(vz - 1);
      if (sj >= 0) {
        map[sj * stride] = nent;
        if (sz >= 0) {  // drop the dead zi entry
          --nl;
          if (sz != nl) map[sz * stride] = map[nl * stride];
        }
      } else if (sz >= 0) {
        map[sz * stride] = nent;  // reuse the dead slot
      } else {
        if (nl == cap) {
          emitted += z;
          return false;
        }
        map[nl * stride] = nent;
        ++nl;
      }
    } else if (sz >= 0) {
      --nl;
      if (sz != nl) map[sz * stride] = map[nl * stride];
    }
    if (reg_min<kSharedRegs>(&regs[vj - 1], (u64)__double_as_longlong(t), id))
      atomicSub(unset_ctr, 1);
  }
  emitted += z;
  return true;
}

// ---- warp walker ----------------------------------------------------------
// Dense view of an element's permutation: k words, entry (stamp << 16) |
// (val - 1); words with another stamp read as the identity.  The array is a
// plain k-word slice (global scratch) or a strided region of shared memory
// (the owning warp's lane tables, see gm_csr.cuh).
struct DenseFlat {
  u32* p;
  __device__ __forceinline__ u32& operator[](u32 i) const { return p[i]; }
};
template <class D>
__device__ __forceinline__ auto dload(const D& d, u32 i) { return d[i]; }
template <class D, class V>
__device__ __forceinline__ void dstore(const D& d, u32 i, V v) { d[i] = v; }
template <class D>
struct DenseWord { typedef std::remove_cv_t<std::remove_reference_t<decltype(std::declval<D>()[0])>> type; };

struct DenseStrided {  // 128-word rows, `pitch` words apart
  u32* p;
  u32 pitch;
  __device__ __forceinline__ u32& operator[](u32 i) const { return p[(i >> 7) * pitch + (i & 127u)]; }
};

template <class D>
__device__ __forceinline__ u32 dget(const D& dense, u32 pos, u32 stamp) {
  typedef typename DenseWord<D>::type W;
  if (!FyWord<W>::BIG && !GM_OKIF(pos < 65536u, 20u)) return pos + 1;
  const W e = dload(dense, pos);
  return (u32)(e >> FyWord<W>::SH) == stamp ? (u32)(e & FyWord<W>::LOW) + 1 : pos + 1;
}

// One element, 32 queue steps per iteration.  Resumes at (z_start accepted
// arrivals, b_start = time of the last one); the caller has loaded the live
// permutation entries into `dense`.  scan: 32 doubles, prov: 32 ints (per-warp
// shared scratch).  mtab: Barrett constants of m = k - z + 1 for z < mtab_n
// (nullable).  unset_ctr: decremented when a register is first set (nullable).
// ltab: the log table (the shared-memory copy in K1, the global one in K2).
// fast: every spacing divide of the element may use the branch-free divide
// (w_fast(w)); a run-time flag, so one copy of the walker serves both
// (kernel code size: the K1 kernel keeps its hot loops in the instruction
// cache).
template <bool kSharedRegs, class D>
__device__ __forceinline__ void walk_warp(u64 id, double w, double tau, u32 k, u64 useed,
                                          u64 pseed, const D& dense, u32 stamp, double* scan,
                                          int* prov, Reg* regs, int* unset_ctr, u32& emitted,
                                          u32 z_start = 0, double b_start = 0.0,
                                          const u32* mtab = nullptr, u32 mtab_n = 0,
                                          const double* ltab = &gm_glog_tab[0][0], bool fast = false) {
  const unsigned FULL = 0xFFFFFFFFu;
  const int lane = threadIdx.x & 31;
  const u64 ubase = useed + id * K_ELEM;
  const u64 pbase = pseed + id * K_ELEM;
  double b = b_start;
  u32 z0 = z_start;
  typedef typename DenseWord<D>::type DW;
  while (z0 < k) {
#ifdef GM_STATS_WALK
    long long tw0 = clock64();
#endif
    const u32 z = z0 + lane + 1;
    const bool valid = z <= k;
    // the permutation draws and the dense-array reads first (they do not
    // depend on the arrival times): the reads, L1/L2 round trips, then
    // complete under the spacings and the prefix instead of after them
    u32 j = 0;
    if (valid) j = FyWord<DW>::BIG ? perm_draw_big(pbase, z, k)
                   : (mtab && z < mtab_n) ? perm_draw_m(pbase, z, k, mtab[z]) : perm_draw(pbase, z, k);
    const u32 zi = z - 1, ji = j - 1;
    // raw words only: they are decoded after the spacings and the prefix, so
    // the warp does not wait for the loads before its arithmetic
    DW ez = 0, ej = 0;
    if (valid && (FyWord<DW>::BIG || GM_OKIF(ji < 65536u, 20u))) {
      ez = dload(dense, zi);
      ej = dload(dense, ji);
    }
    double d = 0.0;
    if (valid) {
      const u64 x = mix64(ubase + (u64)z * K_STEP);
      const double L = -log_pos_t(u_open(x), ltab);  // ltab: shared memory (K1) or the global copy (K2)
      const double D = __dmul_rn(w, (double)(k - z + 1));
      d = fast ? ddiv_fast(L, D) : ddiv_ieee(L, D);
    }
#ifdef GM_STATS_WALK
    { const long long tw1 = clock64(); if (lane == 0) atomicAdd(&g_stats[5], (unsigned long long)(tw1 - tw0)); tw0 = tw1; }
#endif
    scan[lane] = d;
    prov[lane] = -1;
    __syncwarp();
    if (lane == 0) {  // left-to-right prefix, the reference's summation order
      double2* s2 = reinterpret_cast<double2*>(scan);
      double2 v[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = s2[i];
      double acc = b;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        acc = __dadd_rn(acc, v[i].x);
        v[i].x = acc;
        acc = __dadd_rn(acc, v[i].y);
        v[i].y = acc;
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) s2[i] = v[i];
    }
    __syncwarp();
#ifdef GM_STATS_WALK
    { const long long tw1 = clock64(); if (lane == 0) atomicAdd(&g_stats[6], (unsigned long long)(tw1 - tw0)); tw0 = tw1; }
#endif
    const double t = scan[lane];
    u32 vz = valid ? ((u32)(ez >> FyWord<DW>::SH) == stamp ? (u32)(ez & FyWord<DW>::LOW) + 1 : zi + 1) : 0u;
    const u32 mj = valid ? ((u32)(ej >> FyWord<DW>::SH) == stamp ? (u32)(ej & FyWord<DW>::LOW) + 1 : ji + 1) : 0u;
    const u32 stop = __ballot_sync(FULL, !(valid && t <= tau));
    const int n_acc = stop ? __ffs(stop) - 1 : 32;
    const bool acc = lane < n_acc;
    // provider of position zi: last earlier lane whose ji == zi
    const int tgt = (int)ji - (int)z0;
    if (acc && tgt > lane && tgt < n_acc) atomicMax(&prov[tgt], lane);
    __syncwarp();
    int p = acc ? prov[lane] : -1;
    // provider of position ji: last earlier lane with the same ji
    const u32 same = __match_any_sync(FULL, acc ? ji : (0x80000000u | (u32)lane));
    const u32 lower = same & ((1u << lane) - 1u);
    const int pj = lower ? 31 - __clz(lower) : -1;
    // resolve vz through provider chains (pointer jumping)
    while (__any_sync(FULL, p >= 0)) {
      const int src = p >= 0 ? p : lane;
      const u32 v2 = __shfl_sync(FULL, vz, src);
      const int p2 = __shfl_sync(FULL, p, src);
      if (p >= 0) {
        vz = v2;
        p = p2;
      }
    }
    const u32 vjp = __shfl_sync(FULL, vz, pj >= 0 ? pj : lane);
    const u32 vj = pj >= 0 ? vjp : mj;
    // positions >= z0 + n_acc stay live: last writer of each ji stores vz
    const u32 higher = same & ~((2u << lane) - 1u);
    GM_CHECK(!acc || (vj >= 1 && vj <= k && vz >= 1 && vz <= k && ji < k), 3u);
    if (acc && higher == 0 && ji >= z0 + (u32)n_acc && GM_OKIF(ji < k, 21u))
      dstore(dense, ji, ((DW)stamp << FyWord<DW>::SH) | (DW)(vz - 1));
    if (acc && GM_OKIF(vj >= 1 && vj <= k, 22u) &&
        reg_min<kSharedRegs>(&regs[vj - 1], (u64)__double_as_longlong(t), id) && unset_ctr)
      atomicSub(unset_ctr, 1);
    emitted += (u32)(n_acc + (n_acc < 32 && z0 + n_acc < k ? 1 : 0));
#ifdef GM_STATS_WALK
    { const long long tw1 = clock64(); if (lane == 0) { atomicAdd(&g_stats[7], (unsigned long long)(tw1 - tw0)); atomicAdd(&g_stats[0], 1ull); } }
#endif
    if (n_acc < 32) break;
    b = __shfl_sync(FULL, t, 31);
    z0 += 32;
    __syncwarp();
  }
  __syncwarp();
}

}  // namespace gmk
