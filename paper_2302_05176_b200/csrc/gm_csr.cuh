// gm_csr.cuh -- K1 building blocks: batched FastGM sketches of CSR vectors
// (sm_100a); the kernel itself, csr4_kernel, is in gm_csr4.cuh.
//
// Replaces sketch_fast_counted (sketch.py:218-311) applied to every vector
// of a batch.  Each vector is sketched by threshold passes (DESIGN.md
// section 3): every arrival t <= tau of every element queue (_run_queue,
// randgen.py:158-207) is folded into the k registers; a pass that leaves a
// register unset is repeated with a larger tau.
//
// Lane walker: one lane walks one element, one queue step per call
// (straight-line step: the next spacing, the permutation draw, the lane's
// Fisher-Yates lookup, the register read; rare cases take a slow path).
// k <= 1024: lane_step_log, the lane's Fisher-Yates state is its draw log and
// a bit map of drawn positions (below); larger k: lane_step, a per-lane
// (position, value) table.  An element whose expected depth k*w*tau is
// large, or whose log / table fills up, is walked by the whole warp in-line
// (walk_warp, 32 steps per iteration).
//
// Vector slots: the CTA keeps V vectors in flight (k registers in shared
// memory + a header, SlotInfo); slot_load takes the next vector of the batch
// into a slot (its weight sum, validation and divide-range check in the same
// warp pass), slot_open_pass (re)opens a pass with its tau.
//
// Lane permutation table (k > 1024; LazyPermutation, randgen.py:146-155): NB buckets of
// 4 words per lane, open addressing with bucket-linear probing, cleared when
// the lane takes an element; a word is (position << 16) | (value - 1), 0 =
// empty (a stored position is some j - 1 >= z >= 1).  Entries are never
// removed (an entry below the current step is dead and never looked up
// again).  Layout is bucket-major ((bucket * NT + lane) * 4 + way) so a
// warp's LDS.128 touch distinct bank quads per quarter-warp.
#pragma once

#include "gm_kernels.cuh"

namespace gmk {

#ifndef GM_U
#define GM_U 4
#endif

template <int NT_, int NB_, int V_ = 2, int MINB_ = 1, int DEEP_PCT_ = 62, int DRAIN_LIVE_ = 0, int PB_ = 16,
          int WQ_ = 0, int QCAP_ = 64>
struct CsrCfg {
  // WQ > 0: elements reach the lanes through a per-warp queue instead of
  // per-lane tickets: the warp takes WQ tickets at a time, stages their ids
  // and weights in shared memory (cp.async, in flight during a round of lane
  // steps), tests every element's first arrival against the pass's tau with
  // the K2 filter's exact-safe fp32 bound, counts the ones that cannot reach
  // tau as finished (one arrival each) and queues the rest for the lanes
  static constexpr int WQ = WQ_;
  static constexpr int QCAP = WQ_ > 0 ? QCAP_ : 1;  // queued survivors per warp (ring; the test of a
                                                     // staged batch pauses while the ring is full)
  static_assert(WQ_ == 0 || (QCAP_ >= 32 && WQ_ % 32 == 0), "WQ: whole warps of tickets, ring >= 32");
  static constexpr int DRAIN_LIVE = DRAIN_LIVE_;  // queue empty and <= this many live lanes: warp-walk them
  static constexpr int NT = NT_;               // threads per CTA
  static constexpr int NWARP = NT_ / 32;
  static constexpr int MINB = MINB_;           // __launch_bounds__ min blocks
  static constexpr int NB = NB_;               // buckets per lane table (power of 2); draw-log mode: log words / 2
  // words per lane: the table, or (draw-log mode) the bit map + the draw log
  static constexpr int SLOTS = PB_ <= 10 ? (1 << PB_) / 32 + 2 * NB_ : 4 * NB_;
  // inserts (draw-log mode: logged steps, 4 * NB_) per element before hand-over
  static constexpr int CAPI = (PB_ <= 10 ? 4 * NB_ : 4 * NB_) * 13 / 16;
  static constexpr int V = V_;                 // vectors in flight per CTA
  static constexpr int U = GM_U;               // lane steps per loop iteration
  static constexpr int MTAB = 256;             // Barrett table entries (z < MTAB)
  static constexpr int NMAX = (1 << 24) - 4096;  // elements per vector
  // lane-table word: position and value - 1 in PB bits each; PB = 12 (k <=
  // 4096) leaves the top 8 bits for the element's generation tag, so a lane
  // starting an element retires the previous one's entries by bumping its
  // tag instead of clearing the table (PB = 16: no tag, cleared per element)
  static constexpr int PB = PB_;
  static constexpr bool GEN = PB_ < 16;
  static constexpr u32 VMASK = (1u << PB_) - 1u;
  static constexpr u32 KMAX = 1u << PB_;       // largest k this configuration serves
  // PB = 10 (k <= 1024): draw-log mode.  The lane keeps no (position, value)
  // table: a k-bit map of the positions drawn so far (the first SLOTS / 2
  // words of the lane's area, bucket-major like the table) and the raw draws
  // of its steps in order (16-bit entries in the other half, word-major).  A
  // draw whose bit is clear hits an untouched position (value = position + 1,
  // the common case: one LDS.32, no probe); a set bit is resolved by tracing
  // the draw log backwards (log_trace), exactly
  static constexpr bool LOGM = PB_ <= 10;
  static constexpr int BMW = (1 << PB_) / 32;  // LOGM: bit-map words per lane (KMAX bits)
  static constexpr int BMB = (BMW + 3) / 4;    // LOGM: bit-map buckets (4 words each)
  static constexpr int LOGCAP = 4 * NB_;       // LOGM: logged steps per element (2 per word) before hand-over
  static_assert(PB_ > 10 || PB_ >= 7, "draw-log mode: whole bit-map buckets");
  // expected depth at which an element goes straight to the warp walker
  static constexpr double kDeep = CAPI * (DEEP_PCT_ / 100.0);
  static_assert(PB_ <= 10 || (NB_ & (NB_ - 1)) == 0, "NB must be a power of two");
  static_assert(V_ >= 1 && V_ <= 8, "1..8 slots");
  // per-slot field width of a lane's packed finished-element counts
  static constexpr int FW = V_ <= 4 ? 8 : V_ <= 5 ? 6 : 4;
  static_assert(PB_ <= 10 || PB_ == 12 || PB_ == 16, "draw log, 12-bit (tagged) or 16-bit lane-table words");
};

constexpr int SLOT_EMPTY = 0, SLOT_ACTIVE = 1;

struct SlotInfo {
  long long v;             // vector index
  long long lo;            // first CSR position
  double W;                // total weight (sets tau only)
  double tau;              // pass threshold
  double deep_w;           // weight at which an element is warp-walked
  unsigned long long emitted;
  u64 useed, pseed;         // the vector's uniform / permutation stream seeds
  u64 pdelta;               // pseed - useed (an element's permutation base from its uniform base)
  // tickets: grab = (gen << 24) | next element index, hdr = (gen << 24) | n,
  // gen counting the slot's passes.  hdr is published before grab, so a
  // ticket is valid iff its gen matches hdr's and its index is below hdr's n
  // (a ticket of an earlier pass can never validate against a later header)
  alignas(8) unsigned grab;  // (grab, hdr): one 8-byte load
  unsigned hdr;
  unsigned gen;
  int n;                   // elements
  int done;                // completed elements of this pass
  int attempt;
  int state;
  int fast;                // every weight in the branch-free divide's range
  unsigned seq;            // load order (older slots are drained first)
};

struct CsrShared {
  SlotInfo slot[8];
  unsigned seq;
  int cur;                  // the slot lanes take tickets from first (a hint, see take_next)
  // one vector under many seeds: its weight sum, divide range and validity
  // are the same for every sketch -- computed by the first slot load, reused
  double one_W;
  int one_fast, one_state;  // one_state: 0 unknown, 1 valid, 2 invalid weights
};

template <class C>
__host__ __device__ constexpr size_t csr_smem_bytes(u32 k) {
  return (size_t)C::V * k * sizeof(Reg)               // registers of the slots
         + (size_t)C::NT * C::SLOTS * 4              // lane tables
         + (size_t)C::MTAB * 4                       // Barrett table
         + 128 * 16                                  // log table copy
         + (size_t)C::NWARP * 32 * (8 + 4)           // warp-walker scan + prov
         + (size_t)C::MTAB * 8                       // 64-bit Barrett table
         + (C::WQ > 0 ? (size_t)C::NWARP * (8 + C::WQ * 16 + C::QCAP * 20) : 0);  // WQ: ring positions,
                                                                                // staging, ring
}

// ---- lane table ----------------------------------------------------------
template <class C>
__device__ __forceinline__ uint4 tab_bucket(const u32* tab, u32 b) {
  return *reinterpret_cast<const uint4*>(tab + b * (C::NT * 4));
}

// word of the current element: g24 = its generation << 24 (0 when PB = 16)
template <class C>
__device__ __forceinline__ u32 tab_key(u32 p, u32 g24) { return g24 | (p << C::PB); }

// a word belongs to the current element (PB = 16: any non-zero word)
template <class C>
__device__ __forceinline__ bool tab_live(u32 e, u32 g24) {
  return C::GEN ? (e ^ g24) < (1u << 24) : e != 0u;
}

// Fast probe of one bucket for key tab_key(p) (p >= 1, or p = 0, whose
// identity value 1 an empty PB = 16 word also yields): xor with the key
// leaves the matching live word (at most one) below 2**PB with the low bits =
// value - 1.  Returns the min over the 4 words (< 2**PB iff found).  Ways
// fill in order within an element, so a bucket is full iff its last word is
// live and the first free way is the number of live words among the first
// three.
__device__ __forceinline__ u32 probe_min(const uint4 q, u32 key) {
  return min(min(q.x ^ key, q.y ^ key), min(q.z ^ key, q.w ^ key));
}
template <class C>
__device__ __forceinline__ u32 first_empty(const uint4 q, u32 g24) {
  return tab_live<C>(q.z, g24) ? 3u : tab_live<C>(q.y, g24) ? 2u : tab_live<C>(q.x, g24) ? 1u : 0u;
}

// Full lookup (slow path): value - 1 at position p (p if absent) | word
// index of its entry << 16 (0x3FFF if absent) | first free word on the probe
// path << 30 (0x3FFF if none).
template <class C>
__device__ __noinline__ u64 tab_find(const u32* tab, u32 p, u32 g24) {
  const u32 key = tab_key<C>(p, g24);
  u32 vm1 = p, slot = 0x3FFFu, fre = 0x3FFFu, b = p & (C::NB - 1);
  for (int it = 0; it < C::NB; ++it) {
    const uint4 q = tab_bucket<C>(tab, b);
    const u32 e[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int wy = 3; wy >= 0; --wy) {
      const bool live = tab_live<C>(e[wy], g24);
      if (live && (e[wy] ^ key) <= C::VMASK) {
        slot = b * 4 + wy;
        vm1 = e[wy] & C::VMASK;
      }
      if (!live) fre = b * 4 + wy;
    }
    if (slot != 0x3FFFu || fre != 0x3FFFu) break;
    b = (b + 1) & (C::NB - 1);
  }
  return (u64)vm1 | ((u64)slot << 16) | ((u64)fre << 30);
}

template <class C>
__device__ __forceinline__ void tab_put(u32* tab, u32 slot, u32 e) {
  tab[(slot >> 2) * (C::NT * 4) + (slot & 3)] = e;
}

template <class C>
__device__ __forceinline__ void tab_clear(u32* tab) {
#pragma unroll
  for (int b = 0; b < C::NB; ++b) *reinterpret_cast<uint4*>(tab + b * (C::NT * 4)) = make_uint4(0, 0, 0, 0);
}

// the lane starts an element: retire the previous element's table entries
// (bump the generation; clear the table when the tag wraps, or always when
// PB = 16)
template <class C>
__device__ __forceinline__ void tab_next_element(u32* tab, u32& g24) {
  if (C::GEN) {
    g24 += 1u << 24;
    if (g24 == 0u) {
      tab_clear<C>(tab);
      g24 = 1u << 24;
    }
  } else {
    tab_clear<C>(tab);
  }
}

// ---- lane walker state -----------------------------------------------------
struct Lane {
  u64 id, ubase, pbase;
  double w, b, t, tau;
  Reg* regs;
  u32 z;
  u32 g24;   // the element's lane-table generation << 24 (PB = 12)
  int used;
  int slot;
  bool fast;
};

// One accepted queue step of the lane's element (or, when fresh, only the
// first arrival).  Returns 0: continue, 1: element finished (first arrival
// beyond tau or queue exhausted), 2: table full (state before the step kept
// for a warp to resume).
template <class C>
__device__ __forceinline__ int lane_step(Lane& L, bool fresh, u32* mytab, const u64* mtab64, u32 k,
                                         const double* ltab) {
  const bool acc = !fresh;
  const u32 zs = L.z + 1;
  const u32 g24 = L.g24;
  // permutation draw of step zs and both first-bucket probes
  const u64 g = mix64(L.pbase + (u64)zs * K_STEP);
  const u32 m = k - zs + 1;
  u32 ji = zs - 1 + mod_barrett64(g, m, mtab64[min(zs, (u32)C::MTAB - 1)]);
  const u32 zi = zs - 1;
  u32 bj = ji & (C::NB - 1);
  const u32 kz = tab_key<C>(zi, g24);
  u32 kj = tab_key<C>(ji, g24);
  uint4 qz = tab_bucket<C>(mytab, zi & (C::NB - 1)), qj = tab_bucket<C>(mytab, bj);
  u32 mz = probe_min(qz, kz), mj = probe_min(qj, kj);
  // linear probing continues in the next bucket when the first is full:
  // look there too before falling back to the full lookup (branch-free: when
  // the first bucket settles it, the same bucket is simply read again)
  {
    const u32 nz = ((mz > C::VMASK) & tab_live<C>(qz.w, g24)) ? 1u : 0u;
    const u32 nj = ((mj > C::VMASK) & tab_live<C>(qj.w, g24)) ? 1u : 0u;
    bj = (bj + nj) & (C::NB - 1);
    qz = tab_bucket<C>(mytab, (zi + nz) & (C::NB - 1));
    qj = tab_bucket<C>(mytab, bj);
    mz = probe_min(qz, kz);
    mj = probe_min(qj, kj);
  }
  // next arrival's spacing (independent of this step's permutation work)
  const u32 zn = acc ? min(zs + 1, k) : 1u;
  const u64 x = mix64(L.ubase + (u64)zn * K_STEP);
  const double Lg = -log_pos_t(u_open(x), ltab);
  const double D = __dmul_rn(L.w, (double)(k - zn + 1));
  double dq = ddiv_fast(Lg, D);
  // fast case: no draw rejection, zi resolved in its first bucket, ji found
  // in its first bucket (overwrite) or absent with a free way there (insert)
  const bool jfound = mj <= C::VMASK;
  const bool redraw = ((u32)(g >> 32) == 0xFFFFFFFFu) | (zs >= (u32)C::MTAB);  // the Barrett draw is not exact
  const bool slow = acc & (redraw | ((mz > C::VMASK) & tab_live<C>(qz.w, g24)) |
                           (!jfound & tab_live<C>(qj.w, g24)));
  u32 vz = mz <= C::VMASK ? mz + 1 : zi + 1;
  u32 vj = jfound ? mj + 1 : ji + 1;
  const u32 jway = jfound ? (((qj.x ^ kj) <= C::VMASK) ? 0u : ((qj.y ^ kj) <= C::VMASK) ? 1u
                             : ((qj.z ^ kj) <= C::VMASK) ? 2u : 3u)
                          : first_empty<C>(qj, g24);
  u32 put_slot = bj * 4 + jway;
  bool fresh_slot = !jfound;
  if (!L.fast) dq = ddiv_ieee(Lg, D);
  if (slow) {
    // a full first bucket alone keeps the fast draw; only a rejected draw or a
    // step beyond the Barrett table needs the exact one
    if (redraw) ji = perm_draw(L.pbase, zs, k) - 1;
    kj = tab_key<C>(ji, g24);
    vz = ((u32)tab_find<C>(mytab, zi, g24) & 0xFFFFu) + 1;
    const u64 fj = tab_find<C>(mytab, ji, g24);
    vj = ((u32)fj & 0xFFFFu) + 1;
    const u32 sj = (u32)(fj >> 16) & 0x3FFFu, fr = (u32)(fj >> 30) & 0x3FFFu;
    fresh_slot = sj == 0x3FFFu;
    put_slot = fresh_slot ? fr : sj;
  }
  // accept step zs (branch-lean: the table write and the register update are
  // predicated on acc; only a full table leaves the straight line)
  const bool moved = ji != zi;
  if (acc & moved & !(!fresh_slot || (L.used < C::CAPI && put_slot != 0x3FFFu)))
    return 2;  // table full: hand over before step zs
  if (!moved) vj = vz;
  if (acc & moved) tab_put<C>(mytab, put_slot, kj | (vz - 1));
  L.used += (acc & moved & fresh_slot) ? 1 : 0;
  reg_min_lane(&L.regs[vj - 1], (u64)__double_as_longlong(L.t), L.id, acc);
  L.b = acc ? L.t : L.b;
  L.z = acc ? zs : L.z;
  L.t = __dadd_rn(L.b, dq);
  return (L.z >= k || L.t > L.tau) ? 1 : 0;
}

// ---- draw-log mode (C::LOGM, k <= 1024) --------------------------------------
// The Fisher-Yates state of steps 1..z is the list of their draws j_1..j_z
// (0-based positions).  The content of position p (p >= z) after those steps
// is found by walking the list backwards: a step z' that drew p swapped p's
// content in from position z' - 1, so the trace continues from there (only
// earlier steps can have drawn that position); with no such step left the
// content is still the identity, position + 1.  Equal to LazyPermutation's
// lookup (randgen.py:146-155), with no value ever stored.
//
// lg: the lane's log, word wi at lg[wi * NT], entries 2 wi (low half) and
// 2 wi + 1 (high half).  n: logged steps.  Returns value - 1.
template <class C>
__device__ __noinline__ u32 log_trace(const u32* lg, u32 pos, u32 n) {
  int i = (int)n - 1;
  if (i >= 0 && !(i & 1)) {  // a lone low half at the top
    if ((lg[(i >> 1) * C::NT] & 0xFFFFu) == pos) pos = (u32)i;
    --i;
  }
  for (; i >= 1; i -= 2) {
    const u32 wv = lg[(i >> 1) * C::NT];
    if ((wv >> 16) == pos) pos = (u32)i;
    if ((wv & 0xFFFFu) == pos) pos = (u32)i - 1u;
  }
  return pos;
}

// the lane starts an element: clear the bit map (the log needs no clearing).
// All of the configuration's buckets, whatever k: unconditional stores are
// cheaper than a predicate per bucket.
template <class C>
__device__ __forceinline__ void bm_clear(u32* mybm) {
#pragma unroll
  for (int b = 0; b < C::BMB; ++b) *reinterpret_cast<uint4*>(mybm + b * (C::NT * 4)) = make_uint4(0, 0, 0, 0);
}

// lane_step in draw-log mode (same contract; 2 = the log is full)
template <class C>
__device__ __forceinline__ int lane_step_log(Lane& L, bool fresh, u32* mybm, u32* mylog, const u64* mtab64, u32 k,
                                             const double* ltab) {
  const bool acc = !fresh;
  const u32 zi = L.z, zs = zi + 1;
  if (acc & (zi >= (u32)C::LOGCAP)) return 2;  // hand over before step zs
  // permutation draw of step zs and its bit-map word
  const u64 g = mix64(L.pbase + (u64)zs * K_STEP);
  const u32 m = k - zs + 1;
  u32 ji = zi + mod_barrett64(g, m, mtab64[min(zs, (u32)C::MTAB - 1)]);
  GM_CHECK(ji < k && k <= C::KMAX && zi < k, 30u);
  u32* bw = mybm + (ji >> 7) * (C::NT * 4) + ((ji >> 5) & 3u);
  u32 word = *bw;
  // next arrival's spacing (independent of this step's permutation work)
  const u32 zn = acc ? min(zs + 1, k) : 1u;
  const u64 x = mix64(L.ubase + (u64)zn * K_STEP);
  const double Lg = -log_pos_t(u_open(x), ltab);
  const double D = __dmul_rn(L.w, (double)(k - zn + 1));
  double dq = ddiv_fast(Lg, D);
  if (!L.fast) dq = ddiv_ieee(Lg, D);
  const bool redraw = ((u32)(g >> 32) == 0xFFFFFFFFu) | (zs >= (u32)C::MTAB);  // the Barrett draw is not exact
  u32 vj = ji;  // value - 1
  if (acc & (redraw | (((word >> (ji & 31u)) & 1u) != 0u))) {
    if (redraw) {
      ji = perm_draw(L.pbase, zs, k) - 1;
      bw = mybm + (ji >> 7) * (C::NT * 4) + ((ji >> 5) & 3u);
      word = *bw;
    }
    vj = ((word >> (ji & 31u)) & 1u) ? log_trace<C>(mylog, ji, zi) : ji;
  }
  GM_CHECK(!acc || (ji < k && vj < k && zi < (u32)C::LOGCAP), 31u);
  if (acc) {
    *bw = word | (1u << (ji & 31u));
    reinterpret_cast<unsigned short*>(mylog + (zi >> 1) * C::NT)[zi & 1u] = (unsigned short)ji;
  }
  reg_min_lane(&L.regs[vj], (u64)__double_as_longlong(L.t), L.id, acc);
  L.b = acc ? L.t : L.b;
  L.z = acc ? zs : L.z;
  L.t = __dadd_rn(L.b, dq);
  return (L.z >= k || L.t > L.tau) ? 1 : 0;
}

// ---- vector slots ----------------------------------------------------------
template <class C>
__device__ __forceinline__ Reg* slot_regs(unsigned char* smem, int s, u32 k) {
  return reinterpret_cast<Reg*>(smem) + (size_t)s * k;
}

// open a slot for pass `attempt` of its vector (lane 0 writes the header,
// then publishes the grab word).  A ticket taken from the previous pass's word
// carries that pass's n and an index >= n, so it can never validate against
// the new header.
__device__ __forceinline__ void slot_open_pass(SlotInfo& sl, u32 k, int attempt, double kdeep) {
  sl.attempt = attempt;
  sl.tau = pass_tau(sl.W, k, attempt);
  sl.deep_w = kdeep / ((double)k * sl.tau);
  sl.done = 0;
  sl.state = SLOT_ACTIVE;
  const unsigned gen = (sl.gen + 1u) & 0xFFu;
  sl.gen = gen;
  *(volatile unsigned*)&sl.hdr = (gen << 24) | (unsigned)sl.n;
  __threadfence_block();
  atomicExch(&sl.grab, gen << 24);
}

// a ticket t = atomicAdd(&grab, 1) is valid for the pass whose header h
// (read after the atomic) has the same generation and more elements
__device__ __forceinline__ bool ticket_valid(unsigned t, unsigned h) {
  return ((t ^ h) >> 24) == 0u && (t & 0xFFFFFFu) < (h & 0xFFFFFFu);
}

// warp-uniform: take the next vector of the batch into slot s (or mark it
// empty when the batch is exhausted)

//
// Wsum == nullptr: the slot computes the vector's total weight, validates
// its weights and checks the fast-divide range itself (the prep kernel's work
// for this vector, in the same order: the same W), so the batch needs no
// prep launch.
template <class C, class WT>
__device__ __noinline__ void slot_load(CsrShared& S, int s, unsigned char* smem, u32 k, const int64_t* offsets,
                          int64_t n_vec, const double* Wsum, const int* vflags, int* vec_counter,
                          unsigned long long* err, int attempt0, int lane, const int* vec_list,
                          const WT* wts, u64 useed, u64 salt, const u64* vseeds, int one_vec) {
  const unsigned FULL = 0xFFFFFFFFu;
  SlotInfo& sl = S.slot[s];
  for (;;) {
    long long v = 0;
    if (lane == 0) v = atomicAdd(vec_counter, 1);
    v = __shfl_sync(FULL, v, 0);
    if (v >= n_vec) {
      if (lane == 0) {
        sl.state = SLOT_EMPTY;
        const unsigned gen = (sl.gen + 1u) & 0xFFu;
        sl.gen = gen;
        *(volatile unsigned*)&sl.hdr = gen << 24;  // n = 0: no ticket validates
        __threadfence_block();
        atomicExch(&sl.grab, gen << 24);
        __threadfence_block();
      }
      __syncwarp();
      return;
    }
    if (vec_list) v = vec_list[v];  // a subset of the batch (re-runs)
    // one_vec: every sketch of the batch is of the single vector offsets[0..1]
    // (one vector under many seeds, gm_sketch_csr_seeded + GM_FLAG_ONE_VECTOR)
    const int64_t* ov = one_vec ? offsets : offsets + v;
    const int64_t lo = ov[0], n = ov[1] - lo;
    if (n <= 0) {  // EmptyVectorError (latched here without a prep kernel)
      if (!Wsum && lane == 0) atomicCAS(err, 0ull, ((unsigned long long)(v & 0xFFFFFFFF) << 32) | 1u);
      continue;
    }
    if (n > C::NMAX) {
      if (lane == 0) atomicCAS(err, 0ull, ((unsigned long long)(v & 0xFFFFFFFF) << 32) | 3u);
      continue;
    }
    double W = 0.0;
    int fast = 1;
    const int ostate = one_vec ? *(volatile int*)&S.one_state : 0;
    if (ostate == 1) {  // the one vector's sum, computed by an earlier slot load
      __threadfence_block();
      W = *(volatile double*)&S.one_W;
      fast = *(volatile int*)&S.one_fast;
    } else if (ostate == 2) {
      if (lane == 0) atomicCAS(err, 0ull, ((unsigned long long)(v & 0xFFFFFFFF) << 32) | 2u);
      continue;
    } else if (!Wsum) {
      int bad = 0;
      for (int64_t i0 = lo + lane; i0 < lo + n; i0 += 8 * 32) {  // 8 loads in flight per lane
        WT wv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) wv[u] = i0 + u * 32 < lo + n ? __ldcg(&wts[i0 + u * 32]) : WT(0);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (i0 + u * 32 < lo + n) {
            const double w = (double)wv[u];
            bad |= !(isfinite(w) && w > 0.0 && w >= 1e-300);
            fast &= w_fast(w);
            W += w;
          }
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) W += __shfl_xor_sync(FULL, W, o);
      fast = __all_sync(FULL, fast);
      const bool any_bad = __any_sync(FULL, bad);
      if (one_vec && lane == 0) {  // (two first loads may both get here: same values)
        S.one_W = W;
        S.one_fast = fast;
        __threadfence_block();
        *(volatile int*)&S.one_state = any_bad ? 2 : 1;
      }
      if (any_bad) {
        if (lane == 0) atomicCAS(err, 0ull, ((unsigned long long)(v & 0xFFFFFFFF) << 32) | 2u);
        continue;
      }
    }
    Reg* regs = slot_regs<C>(smem, s, k);
    for (u32 j = lane; j < k; j += 32)
      *reinterpret_cast<uint4*>(&regs[j]) = make_uint4((u32)INF_BITS, (u32)(INF_BITS >> 32), 0xFFFFFFFFu, 0xFFFFFFFFu);
    __threadfence_block();
    __syncwarp();
    if (lane == 0) {
      sl.v = v;
      sl.lo = lo;
      sl.n = (int)n;
      sl.W = Wsum ? Wsum[v] : W;
      // per-vector seeds (a batch of one vector under many seeds) or the batch's
      sl.useed = vseeds ? vseeds[v] : useed;
      sl.pseed = sl.useed ^ salt;
      sl.pdelta = sl.pseed - sl.useed;
      sl.fast = Wsum ? (vflags[v] & 1) : fast;
      sl.emitted = 0;
      sl.seq = ++S.seq;
      slot_open_pass(sl, k, attempt0, C::kDeep);
      GM_TRACE((unsigned long long)(v & 0xFFFFFFFF) | ((unsigned long long)attempt0 << 32) |
               ((unsigned long long)blockIdx.x << 48) | ((unsigned long long)s << 60));
    }
    __syncwarp();
    return;
  }
}

// ---- K1 ---------------------------------------------------------------------
// The kernel (csr4_kernel, lane-level element scheduling) is in gm_csr4.cuh.

}  // namespace gmk
