// gm_pairs.cuh -- device-side stream checks for bulk (id, weight) pair
// arrays: the reference's per-item stream_update rules (stream.py:58-78)
// evaluated for all items at once.
//
//   * InvalidWeightError at the first item whose weight is not finite, > 0
//     and >= 1e-300 (stream.py:61-66);
//   * InconsistentWeightError at the first item whose id appeared earlier
//     with a different weight (stream.py:67-73);
//   * skip_duplicates: only the first occurrence of each id is sketched
//     (stream.py:74-78) -- a register no-op for the others, so dropping them
//     changes work, not results.
//
// One open-addressing table keyed by id (linear probing, capacity a power of
// two >= 2n) records the first index of each id (atomicMin).  Pass 1 inserts;
// pass 2 compares every item's weight with its id's first weight, folds the
// first offending indices with atomicMin, and compacts first occurrences.
// Each pass streams the arrays once (HBM-bound) plus one random table access
// per item.
#pragma once

#include "gm_core.cuh"

namespace gmk {

constexpr u64 PAIR_EMPTY = ~0ull;  // empty key; the id 2**64-1 uses the extra slot `cap`

__device__ __forceinline__ u64 pair_slot_find(const u64* keys, u64 mask, u64 id) {
  if (id == PAIR_EMPTY) return mask + 1;
  u64 h = mix64(id ^ 0x5851F42D4C957F2Dull) & mask;
  while (true) {
    const u64 k = __ldcg(&keys[h]);
    if (k == id) return h;
    h = (h + 1) & mask;
  }
}

template <class IdT>
__global__ void __launch_bounds__(256) pairs_insert_kernel(const IdT* __restrict__ ids, int64_t n, u64* keys,
                                                           unsigned long long* first, u64 mask) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const u64 id = (u64)ids[i];
    u64 h;
    if (id == PAIR_EMPTY) {
      h = mask + 1;
    } else {
      h = mix64(id ^ 0x5851F42D4C957F2Dull) & mask;
      while (true) {
        const u64 prev = atomicCAS((unsigned long long*)&keys[h], (unsigned long long)PAIR_EMPTY,
                                   (unsigned long long)id);
        if (prev == PAIR_EMPTY || prev == id) break;
        h = (h + 1) & mask;
      }
    }
    atomicMin(&first[h], (unsigned long long)i);
  }
}

template <class WT>
__device__ __forceinline__ bool pair_weight_ok(WT w) {
  const double d = (double)w;
  return isfinite(d) && d > 0.0 && d >= 1e-300;
}

// out[0] = first invalid-weight index, out[1] = first inconsistent index
// (both start at ~0), out[2] = number of first occurrences written to
// uniq_ids/uniq_w (nullable: checks only)
template <class IdT, class WT>
__global__ void __launch_bounds__(256) pairs_check_kernel(const IdT* __restrict__ ids, const WT* __restrict__ wts,
                                                          int64_t n, const u64* keys,
                                                          const unsigned long long* first, u64 mask,
                                                          unsigned long long* out, IdT* uniq_ids, WT* uniq_w) {
  const int lane = threadIdx.x & 31;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < n; i0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = i0 + threadIdx.x;
    bool lead = false;
    IdT id = 0;
    WT w = 0;
    if (i < n) {
      id = ids[i];
      w = wts[i];
      const u64 h = pair_slot_find(keys, mask, (u64)id);
      const unsigned long long f = __ldcg(&first[h]);
      if (!pair_weight_ok(w)) atomicMin(&out[0], (unsigned long long)i);
      if ((int64_t)f != i && wts[f] != w) atomicMin(&out[1], (unsigned long long)i);
      lead = (int64_t)f == i;
    }
    if (uniq_ids) {  // warp-aggregated compaction of first occurrences
      const unsigned m = __ballot_sync(0xFFFFFFFFu, lead);
      unsigned long long base = 0;
      if (lane == 0 && m) base = atomicAdd(&out[2], (unsigned long long)__popc(m));
      base = __shfl_sync(0xFFFFFFFFu, base, 0);
      if (lead) {
        const unsigned long long pos = base + __popc(m & ((1u << lane) - 1u));
        uniq_ids[pos] = id;
        uniq_w[pos] = w;
      }
    }
  }
}

}  // namespace gmk
