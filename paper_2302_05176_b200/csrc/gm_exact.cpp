// Exact-y finalize (host): re-derive every register's value with the
// reference's own arithmetic.
//
// The device returns, per register j, the winning element s_j (bit-identical
// to the reference's argmin) and its arrival time y_j computed with the
// device log, which can differ from glibc's log by an ulp.
// The reference's y_j is the arrival time of s_j's queue at the order
// statistic whose server is j (randgen.py:158-207 emits (b, perm[z-1]) for
// z = 1..k).  This pass walks each winning element's queue on the host with
// glibc log and IEEE double arithmetic in the reference's operation order
// (u: randgen.py:119; b += -log(u) / (w * (k - z + 1)): :180-187; the
// permutation draw with rejection: :188-199; the lazy Fisher-Yates swap:
// :200-203) until every register it won has been emitted, and stores those
// times: y becomes bit-identical to the reference's.
//
// Cost: one queue walk per distinct winner, up to the largest order
// statistic it holds (tens of steps at the configs' sizes); vectors run in
// parallel on host threads.  Host memory only; no CUDA calls.
//
// Compiled without fast-math and without FMA contraction (-ffp-contract=off)
// so every operation is the IEEE operation CPython performs.

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <utility>
#include <vector>

#include "../../include/gmsketch_b200.h"

namespace {

using u32 = uint32_t;
using u64 = uint64_t;

constexpr u64 kElem = 0x9E3779B97F4A7C15ull;   // randgen.py:46
constexpr u64 kStep = 0xC2B2AE3D27D4EB4Full;   // randgen.py:47
constexpr u64 kRetry = 0xD6E8FEB86659FD93ull;  // randgen.py:48

inline u64 splitmix(u64 x) {  // randgen.py:64-69
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// per-thread scratch: a stamped dense Fisher-Yates array and a stamped
// "wanted server" mark, both of length k
struct Scratch {
  std::vector<u32> perm, perm_stamp, want_stamp;
  u32 pstamp = 0, wstamp = 0;
  explicit Scratch(u32 k) : perm(k), perm_stamp(k, 0), want_stamp(k, 0) {}
  u32 get(u32 pos) const { return perm_stamp[pos] == pstamp ? perm[pos] : pos + 1; }
  void set(u32 pos, u32 v) {
    perm[pos] = v;
    perm_stamp[pos] = pstamp;
  }
  void next_walk() {
    if (++pstamp == 0) {
      std::fill(perm_stamp.begin(), perm_stamp.end(), 0u);
      pstamp = 1;
    }
  }
  void next_group() {
    if (++wstamp == 0) {
      std::fill(want_stamp.begin(), want_stamp.end(), 0u);
      wstamp = 1;
    }
  }
};

// Walk element `id` (weight w) from z = 1 and store the arrival time of every
// server marked wanted; returns false if some wanted server is never reached
// (impossible for a genuine winner: the queue visits every server by z = k).
bool walk_element(Scratch& sc, u64 useed, u64 pseed, u64 id, double w, u32 k, u32 n_want, double* y) {
  sc.next_walk();
  const u64 ubase = useed + id * kElem, pbase = pseed + id * kElem;
  double b = 0.0;
  for (u32 z = 1; z <= k && n_want; ++z) {
    const u64 x = splitmix(ubase + (u64)z * kStep);
    const double u = (double)(x >> 11) * 0x1p-53 + 0x1p-54;
    const u32 mz = k - z + 1;
    const double den = w * (double)mz;
    b = b + (-std::log(u)) / den;
    const u64 m = mz;
    const u64 rem = (UINT64_MAX % m + 1) % m;  // 2**64 mod m
    u64 g = splitmix(pbase + (u64)z * kStep);
    for (u64 a = 1; rem != 0 && g >= (u64)0 - rem; ++a) g = splitmix(pbase + (u64)z * kStep + a * kRetry);
    const u32 jpos = (u32)(z - 1 + g % m);  // 0-based position drawn in [z-1, k-1]
    const u32 vz = sc.get(z - 1), vj = sc.get(jpos);
    sc.set(z - 1, vj);
    sc.set(jpos, vz);
    const u32 server = vj - 1;  // perm[z-1] after the swap, 0-based
    if (sc.want_stamp[server] == sc.wstamp) {
      y[server] = b;
      sc.want_stamp[server] = 0;
      --n_want;
    }
  }
  return n_want == 0;
}

template <class IdT, class WT>
int exact_one(const IdT* ids, const WT* w, int64_t lo, int64_t hi, u32 k, u64 useed, u64 pseed, const u64* s,
              double* y, Scratch& sc, std::vector<std::pair<u64, u32>>& reg, std::vector<u64>& uniq,
              std::vector<double>& wt) {
  reg.resize(k);
  for (u32 j = 0; j < k; ++j) reg[j] = {s[j], j};
  std::sort(reg.begin(), reg.end());
  uniq.clear();
  for (u32 j = 0; j < k; ++j)
    if (uniq.empty() || uniq.back() != reg[j].first) uniq.push_back(reg[j].first);
  // weights of the winners: one scan of the element range
  wt.assign(uniq.size(), -1.0);
  for (int64_t i = lo; i < hi; ++i) {
    const u64 id = (u64)ids[i];
    auto it = std::lower_bound(uniq.begin(), uniq.end(), id);
    if (it != uniq.end() && *it == id && wt[it - uniq.begin()] < 0.0) wt[it - uniq.begin()] = (double)w[i];
  }
  size_t r = 0;
  for (size_t g = 0; g < uniq.size(); ++g) {
    if (wt[g] < 0.0) return GM_ERR_MISMATCHED;  // a register names an id absent from the input
    sc.next_group();
    u32 n_want = 0;
    for (; r < reg.size() && reg[r].first == uniq[g]; ++r) {
      sc.want_stamp[reg[r].second] = sc.wstamp;
      ++n_want;
    }
    if (!walk_element(sc, useed, pseed, uniq[g], wt[g], k, n_want, y)) return GM_ERR_MISMATCHED;
  }
  return GM_OK;
}

template <class IdT, class WT>
int exact_all(const IdT* ids, const WT* w, const int64_t* offsets, int64_t n_vec, u32 k, u64 useed, u64 pseed,
              const u64* s, double* y, int n_threads) {
  std::atomic<int64_t> next{0};
  std::atomic<int> rc{GM_OK};
  std::atomic<int64_t> bad{-1};
  auto worker = [&]() {
    Scratch sc(k);
    std::vector<std::pair<u64, u32>> reg;
    std::vector<u64> uniq;
    std::vector<double> wt;
    for (;;) {
      const int64_t v = next.fetch_add(1);
      if (v >= n_vec || rc.load() != GM_OK) return;
      const int e = exact_one<IdT, WT>(ids, w, offsets[v], offsets[v + 1], k, useed, pseed, s + v * (int64_t)k,
                                       y + v * (int64_t)k, sc, reg, uniq, wt);
      if (e != GM_OK) {
        int expect = GM_OK;
        if (rc.compare_exchange_strong(expect, e)) bad.store(v);
        return;
      }
    }
  };
  int nt = n_threads > 0 ? n_threads : (int)std::max(1u, std::thread::hardware_concurrency());
  nt = (int)std::min<int64_t>(nt, std::max<int64_t>(1, n_vec));
  if (nt == 1) {
    worker();
  } else {
    std::vector<std::thread> pool;
    for (int t = 0; t < nt; ++t) pool.emplace_back(worker);
    for (auto& t : pool) t.join();
  }
  return rc.load();
}

}  // namespace

// One element's queue advanced by `steps` emissions on the host
// (randgen.py:158-207 with a dense Fisher-Yates array, the state of
// ElementQueueState randgen.py:210-271): perm holds the k entries of the
// permutation (1-based values) and is updated in place; t_out/s_out receive
// the emitted (time, server) pairs.  Host memory only.
extern "C" int gm_exact_y(const void* ids, int id_bits, const void* w, int w_bits, const int64_t* offsets,
                          int64_t n_vec, int32_t k, uint64_t global_seed, uint64_t stream_salt,
                          const uint64_t* s, double* y_io, int32_t n_threads) {
  if ((id_bits != 32 && id_bits != 64) || (w_bits != 32 && w_bits != 64) || k < 1 || n_vec < 0)
    return GM_ERR_INVALID_PARAMETER;
  if (n_vec == 0) return GM_OK;
  const u64 useed = global_seed, pseed = global_seed ^ stream_salt;
  const u32 kk = (u32)k;
  if (id_bits == 32 && w_bits == 32)
    return exact_all<u32, float>((const u32*)ids, (const float*)w, offsets, n_vec, kk, useed, pseed, s, y_io, n_threads);
  if (id_bits == 32)
    return exact_all<u32, double>((const u32*)ids, (const double*)w, offsets, n_vec, kk, useed, pseed, s, y_io, n_threads);
  if (w_bits == 32)
    return exact_all<u64, float>((const u64*)ids, (const float*)w, offsets, n_vec, kk, useed, pseed, s, y_io, n_threads);
  return exact_all<u64, double>((const u64*)ids, (const double*)w, offsets, n_vec, kk, useed, pseed, s, y_io, n_threads);
}
