// gm_split.cuh -- K1s: the CSR batch path split into arrival generation and
// Fisher-Yates resolution (sm_100a).
//
// Same result as csr3_kernel (sketch_fast_counted, sketch.py:218-311, per
// vector), different schedule.  The per-lane Fisher-Yates tables of the fused
// lane walker cap it at 16 warps/SM and make every queue step one long
// dependency chain; here the two halves of a queue step run in kernels that
// suit them:
//
//   A1 depth_kernel    one lane per element: the spacings of U steps at a
//                      time as independent chains, summed left to right in
//                      step order (randgen.py:186) until the first arrival
//                      beyond tau -> depth[e] = accepted arrivals.  No shared
//                      tables: occupancy is bound by registers only.
//   scan               exclusive sum of depth -> aoff (cub::DeviceScan).
//   A2 arrival_kernel  the same walk to the known depth, plus the permutation
//                      draw of every accepted step: writes (t, j - 1, e) of
//                      every accepted arrival contiguously per element.
//   B  fy_kernel       a warp takes whole elements and resolves their swaps 32
//                      consecutive arrivals at a time: within a window the
//                      values an earlier step moved are found by provider
//                      chains (as in walk_warp), keyed per element segment;
//                      an element that continues into the next window carries
//                      its live positions in a stamped dense array.  Every
//                      arrival is folded into its register in global memory
//                      (128-bit CAS, lexicographic (y, id) minimum).
//
// The sketch registers of the batch live in global memory (n_vec x k x 16 B,
// L2 resident for config 2); finalize_kernel writes y/s and lists the vectors
// whose pass left a register unset (the caller re-runs those with a larger
// tau through csr3_kernel).
#pragma once

#include "gm_kernels.cuh"

namespace gmk {

constexpr int SPLIT_NT = 256;

// element -> vector index (one warp per vector)
__global__ void vec_of_kernel(const int64_t* __restrict__ offsets, int64_t n_vec, u32* __restrict__ vec_of) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = gw; v < n_vec; v += nw)
    for (int64_t i = offsets[v] + lane; i < offsets[v + 1]; i += 32) vec_of[i] = (u32)v;
}

__global__ void regs_init_kernel(Reg* __restrict__ r, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    r[i].y = INF_BITS;
    r[i].id = NO_ID;
  }
}

// Warp element feeder: lanes that need an element take the next indices of
// the warp's current chunk; chunks of 32 elements come from a global counter.
struct Feeder {
  long long next, end;  // warp-uniform
  bool done;
};

__device__ __forceinline__ long long feed(Feeder& F, bool need, int64_t n, unsigned long long* counter) {
  const unsigned FULL = 0xFFFFFFFFu;
  const int lane = threadIdx.x & 31;
  long long mine = -1;
  unsigned m = __ballot_sync(FULL, need);
  while (m && !F.done) {
    if (F.next >= F.end) {
      long long c = 0;
      if (lane == 0) c = (long long)atomicAdd(counter, 32ull);
      c = __shfl_sync(FULL, c, 0);
      if (c >= n) {
        F.done = true;
        break;
      }
      F.next = c;
      F.end = min((long long)n, c + 32);
    }
    const int take = (int)min((long long)__popc(m), F.end - F.next);
    const int rank = __popc(m & ((1u << lane) - 1u));
    if (((m >> lane) & 1u) && rank < take) mine = F.next + rank;
    F.next += take;
    m = __ballot_sync(FULL, need && mine < 0);
  }
  return mine;
}

// A1 (kWrite = false): depth[e] = number of arrivals t <= tau_v of element e.
// A2 (kWrite = true):  the depth[e] accepted arrivals (t, j - 1, e) written at
//                      aoff[e] ...
template <class IdT, class WT, bool kWrite>
__global__ void __launch_bounds__(SPLIT_NT)
    arrivals_kernel(const IdT* __restrict__ ids, const WT* __restrict__ wts, int64_t n,
                    const u32* __restrict__ vec_of, const double* __restrict__ Wsum,
                    const int* __restrict__ vflags, u32 k, u64 useed, u64 pseed, int attempt,
                    u32* __restrict__ depth, const unsigned long long* __restrict__ aoff,
                    unsigned long long cap, double* __restrict__ arr_t, unsigned short* __restrict__ arr_j,
                    u32* __restrict__ arr_e, unsigned long long* counter) {
  constexpr int U = 4;
  constexpr int MT = 256;
  __shared__ u32 mtab[MT];
  for (u32 z = threadIdx.x; z < (u32)MT; z += blockDim.x) mtab[z] = (z >= 1 && z <= k) ? barrett_magic(k - z + 1) : 0u;
  __syncthreads();
  const unsigned FULL = 0xFFFFFFFFu;
  Feeder F{0, 0, false};
  long long e = -1;
  u64 ub = 0, pb = 0;
  double w = 0.0, tau = 0.0, b = 0.0;
  u32 z = 0, d = 0;
  unsigned long long off = 0;
  bool fast = true;
  for (;;) {
    const long long ne = feed(F, e < 0, n, counter);
    if (ne >= 0) {
      e = ne;
      w = (double)__ldg(&wts[e]);
      const u64 id = (u64)__ldg(&ids[e]);
      const u32 v = __ldg(&vec_of[e]);
      tau = pass_tau(__ldg(&Wsum[v]), k, attempt);
      fast = (__ldg(&vflags[v]) & 1) != 0;
      ub = useed + id * K_ELEM;
      pb = pseed + id * K_ELEM;
      b = 0.0;
      z = 0;
      if (kWrite) {
        d = depth[e];
        off = aoff[e];
        if (d == 0 || off + d > cap) e = -1;  // nothing to write (or no room: caller re-runs)
      }
    }
    if (!__any_sync(FULL, e >= 0)) {
      if (F.done) break;
      continue;
    }
    if (e < 0) continue;
    // spacings (and draws) of steps z+1..z+U as independent chains
    double sp[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const u32 zu = min(z + 1 + (u32)u, k);
      sp[u] = fast ? spacing_t<true>(ub, zu, w, k) : spacing_t<false>(ub, zu, w, k);
    }
    u32 jd[U];
    if (kWrite) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const u32 zu = min(z + 1 + (u32)u, k);
        jd[u] = zu < (u32)MT ? perm_draw_m(pb, zu, k, mtab[zu]) : perm_draw(pb, zu, k);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (e < 0) break;
      const u32 zs = z + 1;
      if (kWrite) {
        const double t = __dadd_rn(b, sp[u]);
        const unsigned long long a = off + z;
        arr_t[a] = t;
        arr_j[a] = (unsigned short)(jd[u] - 1);
        arr_e[a] = (u32)e;
        b = t;
        z = zs;
        if (z >= d) e = -1;
      } else {
        const double t = __dadd_rn(b, sp[u]);
        if (zs > k || t > tau) {
          depth[e] = z;
          e = -1;
        } else {
          b = t;
          z = zs;
        }
      }
    }
  }
}

// B: Fisher-Yates resolution and register updates, 32 arrivals per window.
template <class IdT>
__global__ void __launch_bounds__(SPLIT_NT)
    fy_kernel(const IdT* __restrict__ ids, int64_t n, const u32* __restrict__ vec_of,
              const unsigned long long* __restrict__ aoff, const double* __restrict__ arr_t,
              const unsigned short* __restrict__ arr_j, const u32* __restrict__ arr_e, u32 k,
              Reg* __restrict__ gregs, u32* __restrict__ dense_global, unsigned long long* counter) {
  __shared__ int prov_all[SPLIT_NT];
  const unsigned FULL = 0xFFFFFFFFu;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int* prov = prov_all + warp * 32;
  u32* dense = dense_global + ((size_t)blockIdx.x * (SPLIT_NT / 32) + warp) * k;
  for (u32 i = lane; i < k; i += 32) dense[i] = 0;
  __syncwarp();
  u32 stamp = 0;
  const unsigned lt = (1u << lane) - 1u;
  for (;;) {
    // a chunk of 32 whole elements
    long long c = 0;
    if (lane == 0) c = (long long)atomicAdd(counter, 32ull);
    c = __shfl_sync(FULL, c, 0);
    if (c >= n) break;
    const long long ce = min((long long)n, c + 32);
    const unsigned long long a_begin = aoff[c], a_end = aoff[ce];
    long long carry_e = -1;  // element whose live positions are in `dense`
    for (unsigned long long base = a_begin; base < a_end; base += 32) {
      const unsigned long long a = base + lane;
      const bool valid = a < a_end;
      const u32 e = valid ? arr_e[a] : 0xFFFFFFFFu;
      const u32 ji = valid ? (u32)arr_j[a] : 0u;
      const double t = valid ? arr_t[a] : 0.0;
      const u32 z = valid ? (u32)(a - aoff[e]) + 1 : 0u;  // queue step of this arrival
      const u32 zi = z - 1;
      const u32 e0 = __shfl_sync(FULL, e, 0);
      const u32 seg = valid ? e - e0 : 31u;  // element segment within the window (< 32)
      const bool carried = valid && (long long)e == carry_e;
      // provider of position zi: last earlier lane of the same element whose
      // ji == zi (that lane is zi - zi_p lanes before this one: steps of one
      // element sit in consecutive lanes)
      prov[lane] = -1;
      __syncwarp();
      const int tgt = lane + (int)min(ji - zi, 32u);
      const u32 e_tgt = __shfl_sync(FULL, e, tgt & 31);
      if (valid && ji > zi && tgt < 32 && e_tgt == e) atomicMax(&prov[tgt], lane);
      __syncwarp();
      int p = valid ? prov[lane] : -1;
      // provider of position ji: last earlier lane of the same element with the same ji
      const u32 same = __match_any_sync(FULL, valid ? ((seg << 16) | ji) : (0x80000000u | (u32)lane));
      const u32 lower = same & lt;
      const int pj = lower ? 31 - __clz(lower) : -1;
      // values before the window: the carried element's dense array, else identity
      u32 vz = zi + 1, mj = ji + 1;
      if (carried) {
        const u32 dz = dense[zi], dj = dense[ji];
        if ((dz >> 16) == stamp) vz = (dz & 0xFFFFu) + 1;
        if ((dj >> 16) == stamp) mj = (dj & 0xFFFFu) + 1;
      }
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
      u32 vj = pj >= 0 ? vjp : mj;
      if (ji == zi) vj = vz;
      // the last element of the window continues into the next window?
      const u32 last_lane = (u32)min(31ull, a_end - 1 - base);
      const u32 e_last = __shfl_sync(FULL, e, last_lane);
      const u32 z_last = __shfl_sync(FULL, z, last_lane);
      const bool cont = base + 32 < a_end && __ldg(&arr_e[base + 32]) == e_last;
      if (cont && (long long)e_last != carry_e) {  // a new element starts carrying: new stamp
        if (++stamp > 0xFFFFu) {
          __syncwarp();
          for (u32 i = lane; i < k; i += 32) dense[i] = 0;
          stamp = 1;
        }
      }
      __syncwarp();
      // carry-out: the last writer of each live position of the continuing element
      const u32 higher = same & ~((2u << lane) - 1u);
      if (cont && valid && e == e_last && ji != zi && higher == 0 && ji >= z_last)
        dense[ji] = (stamp << 16) | (vz - 1);
      carry_e = cont ? (long long)e_last : -1;
      // register update
      if (valid) {
        const u32 v = __ldg(&vec_of[e]);
        reg_min<false>(&gregs[(size_t)v * k + (vj - 1)], (u64)__double_as_longlong(t), (u64)__ldg(&ids[e]));
      }
      __syncwarp();
    }
  }
  // leave the dense scratch clean for other users
  __syncwarp();
  for (u32 i = lane; i < k; i += 32) dense[i] = 0;
}

// y/s out, list of vectors with an unset register (re-run with a larger tau)
__global__ void finalize_kernel(const Reg* __restrict__ gregs, int64_t n_vec, u32 k, double* __restrict__ y_out,
                                u64* __restrict__ s_out, int* __restrict__ redo, int* __restrict__ n_redo) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = gw; v < n_vec; v += nw) {
    bool unset = false;
    for (u32 j = lane; j < k; j += 32) {
      const Reg r = gregs[(size_t)v * k + j];
      unset |= r.y == INF_BITS;
      y_out[(size_t)v * k + j] = __longlong_as_double((long long)r.y);
      s_out[(size_t)v * k + j] = r.id;
    }
    if (__any_sync(0xFFFFFFFFu, unset) && lane == 0) redo[atomicAdd(n_redo, 1)] = (int)v;
  }
}

// executed arrivals per vector (accepted + the terminating one), the
// *_counted work figure
__global__ void split_emitted_kernel(const int64_t* __restrict__ offsets, int64_t n_vec, const u32* __restrict__ depth,
                                     u32 k, int64_t* __restrict__ emitted_out) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = gw; v < n_vec; v += nw) {
    unsigned long long s = 0;
    for (int64_t i = offsets[v] + lane; i < offsets[v + 1]; i += 32) s += depth[i] + (depth[i] < k ? 1u : 0u);
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, o);
    if (lane == 0) emitted_out[v] = (int64_t)s;
  }
}

}  // namespace gmk
