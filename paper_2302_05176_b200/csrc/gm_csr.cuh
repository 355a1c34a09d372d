// gm_csr.cuh -- K1: batched FastGM sketches of CSR vectors (sm_100a).
//
// Replaces sketch_fast_counted (sketch.py:218-311) applied to every vector
// of a batch.  Persistent CTAs; a CTA takes one vector at a time (ticket
// counter), keeps its k registers in shared memory and walks every element's
// queue (_run_queue, randgen.py:158-207) up to a pass threshold tau
// (DESIGN.md section 3).
//
// Work split inside a CTA, per pass and chunk of the vector:
//   1. classify: counting sort of the chunk's elements by expected depth
//      k * w * tau into `order` (deepest first);
//   2. deep elements (expected depth >= C::kDeep) are walked first, one warp
//      per element, 32 queue steps per iteration (walk_warp), with the
//      warp's lane tables reused as the dense permutation array;
//   3. every other element is walked by one lane, one queue step per loop
//      iteration; a lane that finishes takes the next element at once
//      (ids/weights prefetched one element ahead), so lanes never wait for
//      the longest queue of their warp.  The step is straight-line code (the
//      next spacing, the permutation draw, both table probes and the register
//      read), so the compiler interleaves the fp64 and integer chains; rare
//      cases (draw rejection, a full bucket) take a slow path;
//   4. lanes whose permutation table fills up hand the element (z, b, live
//      entries) to a resume record; warps finish those after the lane phase.
//
// Lane permutation table (LazyPermutation, randgen.py:146-155): NB buckets of
// 4 words per lane, open addressing with bucket-linear probing, cleared when
// the lane takes an element; a word is (position << 16) | (value - 1), 0 =
// empty (position 0 is never stored: a stored position is some j - 1 >= z).
// Entries are never removed (an entry below the current step is dead and
// never looked up again).  Layout is bucket-major ((bucket * NT + lane) * 4 +
// way) so a warp's 32 LDS.128 touch 32 distinct bank quads per quarter-warp.
#pragma once

#include "gm_kernels.cuh"

namespace gmk {

template <int NT_, int NB_, int MINB_ = 1>
struct CsrCfg {
  static constexpr int NT = NT_;               // threads per CTA
  static constexpr int NWARP = NT_ / 32;
  static constexpr int MINB = MINB_;           // __launch_bounds__ min blocks
  static constexpr int NB = NB_;               // buckets per lane table (power of 2)
  static constexpr int SLOTS = 4 * NB_;        // words per lane table
  static constexpr int CAPI = SLOTS * 13 / 16; // inserts per element before hand-over
  static constexpr int CHUNK = 1024;           // elements classified at a time
  static constexpr int RCAP = 64;              // resume records per CTA and chunk
  static constexpr int NCLS = 6;               // depth classes
  static constexpr int MTAB = 256;             // Barrett table entries (z < MTAB)
  static constexpr u32 KMAX_REGION = (u32)NB_ * 128u;  // dense array fits the warp's tables
  // expected depth at which an element goes straight to the warp walker
  static constexpr double kDeep = CAPI * 0.62;
  static_assert((NB_ & (NB_ - 1)) == 0, "NB must be a power of two");
};

struct CsrShared {
  int cnt[8];
  int fill[8];
  int deep_grab;
  int lane_grab;
  int n_rec;
  int rec_ovf;
  int vec;
  int fast;
  int pad[2];
  double wsum[32];
};

struct ResumeRec3 {
  u32 elem;  // chunk-local element index
  u32 z;     // accepted arrivals
  u32 nl;    // live entries stored in the record's map slice
  u32 pad;
  double b;  // time of the last accepted arrival
};

template <class C>
__host__ __device__ constexpr size_t csr3_smem_bytes(u32 k) {
  return (size_t)k * sizeof(Reg)                      // registers
         + (size_t)C::NT * C::SLOTS * 4              // lane tables
         + (size_t)C::CHUNK * 4                      // order
         + (size_t)C::MTAB * 4                       // Barrett table
         + (size_t)C::NWARP * 32 * (8 + 4)           // warp-walker scan + prov
         + (size_t)C::RCAP * sizeof(ResumeRec3);     // resume records
}

__device__ __forceinline__ int depth_class(double d, double deep) {
  return d >= deep ? 0 : d >= 16.0 ? 1 : d >= 8.0 ? 2 : d >= 4.0 ? 3 : d >= 2.0 ? 4 : 5;
}

// ---- lane table ----------------------------------------------------------
template <class C>
__device__ __forceinline__ const uint4& tab_bucket(const u32* tab, u32 b) {
  return *reinterpret_cast<const uint4*>(tab + b * (C::NT * 4));
}

// Fast probe of one bucket for position p (p >= 1, or p = 0 whose identity
// value 1 an empty word also yields): xor with p << 16 leaves the matching
// word (at most one) below 2**16 with low half = value - 1.  Returns the min
// over the 4 words (< 2**16 iff found).  Ways fill in order, so a bucket is
// full iff its last word is non-zero and the first empty way is the number
// of non-zero words among the first three.
__device__ __forceinline__ u32 probe_min(const uint4 q, u32 p) {
  const u32 k16 = p << 16;
  return min(min(q.x ^ k16, q.y ^ k16), min(q.z ^ k16, q.w ^ k16));
}
__device__ __forceinline__ u32 first_empty(const uint4 q) {
  return q.z ? 3u : q.y ? 2u : q.x ? 1u : 0u;
}

// Full lookup (slow path): value at position p (identity if absent) packed
// with the word index of its entry (bits 16..29, 0x3FFF if absent) and of the
// first empty word on the probe path (bits 30..43 of the u64, 0x3FFF if none).
template <class C>
__device__ __noinline__ u64 tab_find(const u32* tab, u32 p) {
  u32 val = p + 1, slot = 0x3FFFu, fre = 0x3FFFu, b = p & (C::NB - 1);
  for (int it = 0; it < C::NB; ++it) {
    const uint4 q = *reinterpret_cast<const uint4*>(tab + b * (C::NT * 4));
    const u32 e[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int wy = 3; wy >= 0; --wy) {
      if ((e[wy] >> 16) == p && e[wy] != 0u) {
        slot = b * 4 + wy;
        val = (e[wy] & 0xFFFFu) + 1;
      }
      if (e[wy] == 0u) fre = b * 4 + wy;
    }
    if (slot != 0x3FFFu || fre != 0x3FFFu) break;
    b = (b + 1) & (C::NB - 1);
  }
  return (u64)val | ((u64)slot << 16) | ((u64)fre << 30);
}

template <class C>
__device__ __forceinline__ void tab_put(u32* tab, int slot, u32 e) {
  tab[(slot >> 2) * (C::NT * 4) + (slot & 3)] = e;
}

template <class C>
__device__ __forceinline__ void tab_clear(u32* tab) {
#pragma unroll
  for (int b = 0; b < C::NB; ++b) *reinterpret_cast<uint4*>(tab + b * (C::NT * 4)) = make_uint4(0, 0, 0, 0);
}

// ---- per-CTA context --------------------------------------------------------
template <class C, class IdT, class WT>
struct CsrCtx {
  const IdT* cid;  // chunk ids
  const WT* cw;    // chunk weights
  Reg* regs;
  u32* tables;
  u32* order;
  const u32* mtab;
  double* scan;
  int* prov;
  ResumeRec3* rec;
  u32* rmaps;
  u32* gdense;
  CsrShared* S;
  u32 k;
  u64 useed, pseed;
  double tau;
  int lane, warp, tid;
  bool region_dense;
};

// warp-walker dense array over the warp's table region (cleared on entry and
// on exit, so lane words and dense stamps never meet)
template <class C>
__device__ __forceinline__ void region_clear(u32* tables, int warp, int lane) {
  u32* base = tables + warp * 128 + lane * 4;
#pragma unroll
  for (int b = 0; b < C::NB; ++b) *reinterpret_cast<uint4*>(base + b * (C::NT * 4)) = make_uint4(0, 0, 0, 0);
}

template <class C, class IdT, class WT>
__device__ __forceinline__ void dense_clear(const CsrCtx<C, IdT, WT>& X) {
  if (X.region_dense) region_clear<C>(X.tables, X.warp, X.lane);
  else for (u32 i = X.lane; i < X.k; i += 32) X.gdense[i] = 0;
  __syncwarp();
}

// walk one element with the whole warp, resuming at (z0, b0) with nl live
// entries from `ents` ((pos << 16) | (val - 1)) -- ents may be null
template <class C, class IdT, class WT, bool kFast>
__device__ __forceinline__ void warp_element(const CsrCtx<C, IdT, WT>& X, u32 e, u32 z0, double b0,
                                             const u32* ents, u32 nl, u32& stamp, u32& emitted) {
  if (++stamp > 0xFFFFu) {
    dense_clear(X);
    stamp = 1;
  }
  const DenseStrided dreg{X.tables + X.warp * 128, (u32)(C::NT * 4)};
  const DenseFlat dglob{X.gdense};
  for (u32 i = X.lane; i < nl; i += 32) {
    const u32 ent = ents[i];
    if (X.region_dense) dreg[ent >> 16] = (stamp << 16) | (ent & 0xFFFFu);
    else dglob[ent >> 16] = (stamp << 16) | (ent & 0xFFFFu);
  }
  __syncwarp();
  const u64 id = (u64)__ldg(&X.cid[e]);
  const double w = (double)__ldg(&X.cw[e]);
  u32 em = 0;
  if (X.region_dense)
    walk_warp<true, kFast>(id, w, X.tau, X.k, X.useed, X.pseed, dreg, stamp, X.scan, X.prov, X.regs, nullptr,
                           em, z0, b0, X.mtab, (u32)C::MTAB);
  else
    walk_warp<true, kFast>(id, w, X.tau, X.k, X.useed, X.pseed, dglob, stamp, X.scan, X.prov, X.regs, nullptr,
                           em, z0, b0, X.mtab, (u32)C::MTAB);
  if (X.lane == 0) emitted += em;
}

// ---- one chunk of one pass -----------------------------------------------
template <class C, class IdT, class WT, bool kFast>
__device__ void csr_chunk(const CsrCtx<C, IdT, WT>& X, int cn, u32& emitted) {
  constexpr int NT = C::NT;
  const unsigned FULL = 0xFFFFFFFFu;
  CsrShared& S = *X.S;
  const int lane = X.lane, tid = X.tid;
  const unsigned lt_mask = (1u << lane) - 1u;
  const u32 k = X.k;
  const double tau = X.tau;
  const double kt = (double)k * tau;  // expected depth = k * w * tau

  // (1) classify: counting sort by depth class, deepest first
  if (tid < 8) S.cnt[tid] = 0;
  if (tid == 0) {
    S.deep_grab = 0;
    S.lane_grab = 0;
    S.n_rec = 0;
    S.rec_ovf = 0;
  }
  __syncthreads();
  for (int i0 = 0; i0 < cn; i0 += NT) {
    const int i = i0 + tid;
    const int c = i < cn ? depth_class(kt * (double)__ldg(&X.cw[i]), C::kDeep) : 7;
    const unsigned grp = __match_any_sync(FULL, c);
    if (c < 7 && (grp & lt_mask) == 0) atomicAdd(&S.cnt[c], __popc(grp));
  }
  __syncthreads();
  if (tid == 0) {
    int acc = 0;
    for (int c = 0; c < C::NCLS; ++c) {
      S.fill[c] = acc;
      acc += S.cnt[c];
    }
  }
  __syncthreads();
  const int n_deep = S.cnt[0];
  for (int i0 = 0; i0 < cn; i0 += NT) {
    const int i = i0 + tid;
    const int c = i < cn ? depth_class(kt * (double)__ldg(&X.cw[i]), C::kDeep) : 7;
    const unsigned grp = __match_any_sync(FULL, c);
    const int leader = __ffs(grp) - 1;
    int base = 0;
    if (c < 7 && lane == leader) base = atomicAdd(&S.fill[c], __popc(grp));
    base = __shfl_sync(FULL, base, leader);
    if (c < 7) X.order[base + __popc(grp & lt_mask)] = (u32)i;
  }
  __syncthreads();
  const int n_lane = cn - n_deep;
  u32 stamp = 0;

  // (2) deep elements: one warp each
  if (n_deep > 0) {
    bool began = false;
    for (;;) {
      int q = 0;
      if (lane == 0) q = atomicAdd(&S.deep_grab, 1);
      q = __shfl_sync(FULL, q, 0);
      if (q >= n_deep) break;
      if (!began) {
        if (X.region_dense) dense_clear(X);
        began = true;
      }
      warp_element<C, IdT, WT, kFast>(X, X.order[q], 0u, 0.0, nullptr, 0u, stamp, emitted);
    }
    if (began) {
      __syncwarp();
      dense_clear(X);
      stamp = 0;
    }
  }

  // (3) lane phase
  {
    const u32* lorder = X.order + n_deep;
    u32* mytab = X.tables + tid * 4;
    // prefetched next element (chunk index, id, weight)
    int nq = -1;
    u64 nid = 0;
    double nw = 0.0;
    auto grab = [&](bool want) {
      const unsigned m = __ballot_sync(FULL, want);
      if (!m) return;
      const int leader = __ffs(m) - 1;
      int base = 0;
      if (lane == leader) base = atomicAdd(&S.lane_grab, __popc(m));
      base = __shfl_sync(FULL, base, leader);
      if (want) {
        const int q = base + __popc(m & lt_mask);
        nq = q < n_lane ? (int)lorder[q] : -1;
        if (nq >= 0) {
          nid = (u64)__ldg(&X.cid[nq]);
          nw = (double)__ldg(&X.cw[nq]);
        }
      }
    };
    grab(true);
    bool live = false, fresh = false;
    int cur = -1, used = 0;
    u64 id = 0, ubase = 0, pbase = 0;
    double w = 0.0, b = 0.0, t = 0.0;
    u32 z = 0;
    for (;;) {
      // refill from the prefetched element, then prefetch the next one
      const bool need = !live && nq >= 0;
      if (need) {
        cur = nq;
        id = nid;
        w = nw;
        ubase = X.useed + id * K_ELEM;
        pbase = X.pseed + id * K_ELEM;
        b = 0.0;
        z = 0;
        used = 0;
        tab_clear<C>(mytab);
        live = true;
        fresh = true;
      }
      grab(need);
      if (!__any_sync(FULL, live)) break;
      if (!live) continue;
      // ---- straight-line step: spacing of the next arrival (independent of
      // this step), permutation draw and table probes of step zs = z + 1
      const bool acc = !fresh;
      const u32 zs = z + 1;
      const u32 zn = acc ? min(z + 2, k) : 1u;
      const double dq = spacing_t<kFast>(ubase, zn, w, k);
      const u64 g = mix64(pbase + (u64)zs * K_STEP);
      const u32 m = k - zs + 1, M = X.mtab[min(zs, (u32)C::MTAB - 1)];
      u32 r = mod_barrett((u32)(g >> 32), m, M);
      r = mod_barrett((r << 16) | ((u32)g >> 16), m, M);
      r = mod_barrett((r << 16) | ((u32)g & 0xFFFFu), m, M);
      u32 ji = zs - 1 + r;
      const u32 zi = zs - 1;
      const u32 bz = zi & (C::NB - 1), bj = ji & (C::NB - 1);
      const uint4 qz = tab_bucket<C>(mytab, bz), qj = tab_bucket<C>(mytab, bj);
      const u32 mz = probe_min(qz, zi), mj = probe_min(qj, ji);
      // fast case: no draw rejection, zi resolved in its first bucket, ji absent
      // from the table with a free way in its first bucket
      const bool slow = acc & (((u32)(g >> 32) == 0xFFFFFFFFu) | (zs >= (u32)C::MTAB) |
                               ((mz >= 0x10000u) & (qz.w != 0u)) | (mj < 0x10000u) | (qj.w != 0u));
      u32 vz = mz < 0x10000u ? (mz & 0xFFFFu) + 1 : zi + 1;
      u32 vj = ji + 1;
      u32 put_slot = bj * 4 + first_empty(qj);
      bool fresh_slot = true;
      if (slow) {
        ji = perm_draw(pbase, zs, k) - 1;
        vz = (u32)tab_find<C>(mytab, zi) & 0xFFFFu;
        const u64 fj = tab_find<C>(mytab, ji);
        vj = (u32)fj & 0xFFFFu;
        const u32 sj = (u32)(fj >> 16) & 0x3FFFu, fr = (u32)(fj >> 30) & 0x3FFFu;
        fresh_slot = sj == 0x3FFFu;
        put_slot = fresh_slot ? fr : sj;
      }
      bool ok = true;
      if (acc) {
        if (ji == zi) {
          vj = vz;
        } else if (!fresh_slot || (used < C::CAPI && put_slot != 0x3FFFu)) {
          tab_put<C>(mytab, (int)put_slot, (ji << 16) | (vz - 1));
          used += fresh_slot;
        } else {
          ok = false;
        }
        if (ok) {
          reg_min<true>(&X.regs[vj - 1], (u64)__double_as_longlong(t), id);
          b = t;
          z = zs;
        } else {
          // table full: hand the element (state before step zs) to a warp
          const int rr = atomicAdd(&S.n_rec, 1);
          if (rr < C::RCAP) {
            u32 nl = 0;
            u32* dst = X.rmaps + (size_t)rr * C::SLOTS;
            for (int bk = 0; bk < C::NB; ++bk) {
              const uint4 q = tab_bucket<C>(mytab, bk);
              const u32 ee[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
              for (int wy = 0; wy < 4; ++wy)
                if (ee[wy] != 0u && (ee[wy] >> 16) >= zi) dst[nl++] = ee[wy];
            }
            X.rec[rr].elem = (u32)cur;
            X.rec[rr].z = z;
            X.rec[rr].nl = nl;
            X.rec[rr].b = b;
          } else {
            S.rec_ovf = 1;
          }
          emitted += z;
          live = false;
          continue;
        }
      }
      fresh = false;
      t = __dadd_rn(b, dq);
      if (z >= k || t > tau) {
        emitted += z < k ? z + 1 : z;
        live = false;
      }
    }
  }
  __syncthreads();

  // (4) resumed elements (or, after a record overflow, every lane element)
  const bool all = S.rec_ovf != 0;
  const int nr = all ? n_lane : min(S.n_rec, C::RCAP);
  if (nr > 0) {
    if (tid == 0) S.deep_grab = 0;
    __syncthreads();
    bool began = false;
    for (;;) {
      int q = 0;
      if (lane == 0) q = atomicAdd(&S.deep_grab, 1);
      q = __shfl_sync(FULL, q, 0);
      if (q >= nr) break;
      if (!began) {
        dense_clear(X);
        began = true;
      }
      if (all)
        warp_element<C, IdT, WT, kFast>(X, X.order[n_deep + q], 0u, 0.0, nullptr, 0u, stamp, emitted);
      else
        warp_element<C, IdT, WT, kFast>(X, X.rec[q].elem, X.rec[q].z, X.rec[q].b,
                                        X.rmaps + (size_t)q * C::SLOTS, X.rec[q].nl, stamp, emitted);
    }
    if (began) {
      __syncwarp();
      dense_clear(X);
    }
  }
  __syncthreads();
}

// ---- K1 ---------------------------------------------------------------------
// Dynamic shared memory: Reg regs[k] | u32 tables[NT*SLOTS] | u32 order[CHUNK]
//   | u32 mtab[MTAB] | double scan[NWARP][32] | int prov[NWARP][32] | ResumeRec3 rec[RCAP]
template <class C, class IdT, class WT>
__global__ void __launch_bounds__(C::NT, C::MINB)
    csr3_kernel(const IdT* __restrict__ ids, const WT* __restrict__ wts,
                const int64_t* __restrict__ offsets, int64_t n_vec, u32 k, u64 useed, u64 pseed,
                double* __restrict__ y_out, u64* __restrict__ s_out,
                int64_t* __restrict__ emitted_out, int* __restrict__ vec_counter,
                u32* __restrict__ dense_global, u32* __restrict__ resume_global,
                unsigned long long* __restrict__ err, int attempt0) {
  constexpr int NT = C::NT, NWARP = C::NWARP;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ CsrShared S;
  const unsigned FULL = 0xFFFFFFFFu;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  CsrCtx<C, IdT, WT> X;
  X.regs = reinterpret_cast<Reg*>(smem_raw);
  X.tables = reinterpret_cast<u32*>(smem_raw + (size_t)k * sizeof(Reg));
  X.order = X.tables + (size_t)NT * C::SLOTS;
  u32* mtab = X.order + C::CHUNK;
  X.mtab = mtab;
  double* scan_all = reinterpret_cast<double*>(mtab + C::MTAB);
  int* prov_all = reinterpret_cast<int*>(scan_all + NWARP * 32);
  X.rec = reinterpret_cast<ResumeRec3*>(prov_all + NWARP * 32);
  X.scan = scan_all + warp * 32;
  X.prov = prov_all + warp * 32;
  X.rmaps = resume_global + (size_t)blockIdx.x * C::RCAP * C::SLOTS;
  X.gdense = dense_global ? dense_global + ((size_t)blockIdx.x * NWARP + warp) * k : nullptr;
  X.S = &S;
  X.k = k;
  X.useed = useed;
  X.pseed = pseed;
  X.lane = lane;
  X.warp = warp;
  X.tid = tid;
  X.region_dense = k <= C::KMAX_REGION;

  for (u32 z = tid; z < (u32)C::MTAB; z += NT) mtab[z] = (z >= 1 && z <= k) ? barrett_magic(k - z + 1) : 0u;
  Reg* regs = X.regs;
  __syncthreads();

  for (;;) {
    if (tid == 0) S.vec = atomicAdd(vec_counter, 1);
    __syncthreads();
    const int64_t v = S.vec;
    if (v >= n_vec) break;
    const int64_t lo = offsets[v], hi = offsets[v + 1];
    const int n = (int)(hi - lo);

    // total weight (sets tau only) + validation; registers unset
    double ws = 0.0;
    int fast = 1;
    for (int i = tid; i < n; i += NT) {
      const double w = (double)__ldg(&wts[lo + i]);
      if (!(isfinite(w) && w > 0.0 && w >= 1e-300)) atomicCAS(err, 0ull, ((unsigned long long)(v & 0xFFFFFFFF) << 32) | 2u);
      fast &= w_fast(w);
      ws += w;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) ws += __shfl_xor_sync(FULL, ws, o);
    if (lane == 0) S.wsum[warp] = ws;
    for (u32 j = tid; j < k; j += NT) {
      regs[j].y = INF_BITS;
      regs[j].id = NO_ID;
    }
    if (n == 0 && tid == 0) atomicCAS(err, 0ull, ((unsigned long long)(v & 0xFFFFFFFF) << 32) | 1u);
    fast = __syncthreads_and(fast);
    double W = 0.0;
#pragma unroll
    for (int i = 0; i < NWARP; ++i) W += S.wsum[i];
    u32 emitted = 0;

    for (int attempt = attempt0; n > 0; ++attempt) {
      X.tau = pass_tau(W, k, attempt);
      for (int c0 = 0; c0 < n; c0 += C::CHUNK) {
        X.cid = ids + lo + c0;
        X.cw = wts + lo + c0;
        const int cn = min(C::CHUNK, n - c0);
        if (fast) csr_chunk<C, IdT, WT, true>(X, cn, emitted);
        else csr_chunk<C, IdT, WT, false>(X, cn, emitted);
      }
      // (5) every register set => tau bounded the final maximum: done
      int unset = 0;
      for (u32 j = tid; j < k; j += NT) unset |= regs[j].y == INF_BITS;
      if (!__syncthreads_or(unset)) break;
    }

    if (emitted_out) {
      unsigned long long e = emitted;
#pragma unroll
      for (int o = 16; o; o >>= 1) e += __shfl_xor_sync(FULL, e, o);
      if (lane == 0) S.wsum[warp] = (double)e;
      __syncthreads();
      if (tid == 0) {
        double tot = 0.0;
        for (int i = 0; i < NWARP; ++i) tot += S.wsum[i];
        emitted_out[v] = (int64_t)tot;
      }
    }
    for (u32 j = tid; j < k; j += NT) {
      const Reg r = regs[j];
      y_out[v * (int64_t)k + j] = __longlong_as_double((long long)r.y);
      s_out[v * (int64_t)k + j] = r.id;
    }
    __syncthreads();
  }
}

}  // namespace gmk
