// gm_csr4.cuh -- K1: csr4_kernel, batched FastGM sketches of CSR vectors
// with lane-level element scheduling (configs 1-3; sketch_fast per vector,
// sketch.py:218-311).
//
// Pipelined CTA (no CTA-wide barrier after the prologue): V vector slots
// (gm_csr.cuh); every lane takes its elements itself -- a shared-memory
// ticket on the oldest slot that still has untaken elements -- and keeps its
// NEXT element taken and loading (id, weight from HBM/L2) while it walks the
// current one, so a lane whose element ends goes on with the next one at the
// next step, with no warp-wide hand-out and no idle steps.  A lane starting
// an element clears its bit map of drawn positions (k <= 1024, draw-log lanes)
// or retires its table by bumping a generation tag (k <= 4096), and
// finished elements are counted per warp at the end of each round of lane
// steps (one atomic per slot, the register updates fenced first); the warp
// whose count completes a slot finalises it:
// every register set -> write the sketch out and load the next vector; else
// reopen the slot for the next pass with a larger tau.  Deep elements and
// elements whose draw log / lane table fills up are walked by the whole warp (walk_warp).
// Lane steps run in rounds of u_run steps between the warp-level checks
// (2 / 4 / 6 from the batch's expected arrivals per element).
//
// (Round 1's csr3_kernel handed elements out from a warp queue refilled 32
// entries at a time; lane-level scheduling is 1.65x faster on config 1,
// 1.18x on config 3 and 1.5% on config 2 -- DESIGN.md section 6.)
#pragma once

#include "gm_csr.cuh"

namespace gmk {

// lane steps per scheduling round, by the batch's expected arrivals per
// element (see u_run)
#ifndef GM_URUN0
#define GM_URUN0 2
#endif
#ifndef GM_URUN1
#define GM_URUN1 4
#endif
#ifndef GM_URUN2
#define GM_URUN2 6
#endif

#ifdef GM_WALK_NOINLINE
// the warp walker as a call (kernel code size)
template <class D>
__device__ __noinline__ void csr_walk(u64 id, double w, double tau, u32 k, u64 useed, u64 pseed, const D dense,
                                      u32 stamp, double* scan, int* prov, Reg* regs, u32& emitted, u32 z0,
                                      double b0, const u32* mtab, u32 mtab_n, bool fast) {
  walk_warp<true>(id, w, tau, k, useed, pseed, dense, stamp, scan, prov, regs, nullptr, emitted, z0, b0, mtab,
                  mtab_n, nullptr, fast);
}
#endif

// Dynamic shared memory: Reg regs[V][k] | u32 tables[NB][NT][4] | u32 mtab[MTAB]
//   | double scan[NWARP][32] | int prov[NWARP][32]
// kCount: the caller asked for the per-vector arrival counts (emitted_out);
// the uncounted instantiation carries no count registers or instructions
template <class C, class IdT, class WT, bool kCount>
__global__ void __launch_bounds__(C::NT, C::MINB)
    csr4_kernel(const IdT* __restrict__ ids, const WT* __restrict__ wts,
                const int64_t* __restrict__ offsets, int64_t n_vec, u32 k, u64 useed, u64 salt,
                const u64* __restrict__ vseeds, int one_vec,
                const double* __restrict__ Wsum, const int* __restrict__ vflags,
                double* __restrict__ y_out, u64* __restrict__ s_out,
                int64_t* __restrict__ emitted_out, int* __restrict__ vec_counter,
                u32* __restrict__ dense_global, unsigned long long* __restrict__ err, int attempt0,
                const int* __restrict__ vec_list) {
  constexpr int NT = C::NT, NWARP = C::NWARP, V = C::V;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ CsrShared S;
  const unsigned FULL = 0xFFFFFFFFu;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;

  u32* tables = reinterpret_cast<u32*>(smem_raw + (size_t)V * k * sizeof(Reg));
  u32* mtab = tables + (size_t)NT * C::SLOTS;
  double* ltab = reinterpret_cast<double*>(mtab + C::MTAB);  // 128 x {invc, logc}; 16-byte aligned: MTAB*4 % 16 == 0
  double* scan = ltab + 256 + warp * 32;
  int* prov = reinterpret_cast<int*>(ltab + 256 + NWARP * 32) + warp * 32;
  // floor(2^64 / m) for m = k - z + 1, z < MTAB: the lane step's draw in one 64-bit Barrett reduction
  u64* mtab64 = reinterpret_cast<u64*>(reinterpret_cast<int*>(ltab + 256 + NWARP * 32) + NWARP * 32);
  u32* mytab = tables + tid * 4;
  // draw-log mode: the lane's bit map of drawn positions is the first part of
  // its area (bucket-major, at mytab), its draw log the rest (word-major)
  u32* mylog = tables + (size_t)NT * (C::BMB * 4) + tid;
  // WQ: this warp's staging area (ids, weights of a ticket batch) and queue
  unsigned char* wq_area = reinterpret_cast<unsigned char*>(mtab64 + C::MTAB) + (size_t)warp * (8 + C::WQ * 16 + C::QCAP * 20);
  int* q_pos = reinterpret_cast<int*>(wq_area);  // [0] head, [1] tail: monotone ring positions
  unsigned char* wq_base = wq_area + 8;
  IdT* st_id = reinterpret_cast<IdT*>(wq_base);
  WT* st_w = reinterpret_cast<WT*>(wq_base + C::WQ * 8);
  u64* q_id = reinterpret_cast<u64*>(wq_base + C::WQ * 16);
  double* q_w = reinterpret_cast<double*>(wq_base + C::WQ * 16 + C::QCAP * 8);
  int* q_slot = reinterpret_cast<int*>(wq_base + C::WQ * 16 + C::QCAP * 16);
  u32* dense = dense_global + ((size_t)blockIdx.x * NWARP + warp) * k;

  for (u32 z = tid; z < (u32)C::MTAB; z += NT) {
    mtab[z] = (z >= 1 && z <= k) ? barrett_magic(k - z + 1) : 0u;
    mtab64[z] = (z >= 1 && z <= k) ? barrett_magic64(k - z + 1) : 0ull;
  }
  for (u32 i = tid; i < 256; i += NT) ltab[i] = gm_glog_tab[i >> 1][i & 1];
  if constexpr (C::LOGM)
    bm_clear<C>(mytab);
  else
    tab_clear<C>(mytab);
  if (C::WQ > 0 && lane == 0) q_pos[0] = q_pos[1] = 0;
  for (u32 i = lane; i < k; i += 32) dense[i] = 0;  // stamps restart every launch
  if (tid < V) {
    S.slot[tid].state = SLOT_EMPTY;
    S.slot[tid].n = 0;
    S.slot[tid].grab = 0;
    S.slot[tid].hdr = 0;
    S.slot[tid].gen = 0;
    S.slot[tid].seq = 0;
  }
  if (tid == 0) {
    S.seq = 0;
    S.cur = 0;
    S.one_state = 0;
  }
  __syncthreads();
  if (warp < V)
    slot_load<C, WT>(S, warp, smem_raw, k, offsets, n_vec, Wsum, vflags, vec_counter, err, attempt0, lane, vec_list,
                     wts, useed, salt, vseeds, one_vec);
  __syncthreads();

  Lane L;
  L.z = 0;
  L.used = 0;
  L.slot = 0;
  L.b = L.t = L.tau = L.w = 0.0;
  L.id = L.ubase = L.pbase = 0;
  L.regs = nullptr;
  L.fast = true;
  L.g24 = C::GEN ? 1u << 24 : 0u;
  bool live = false, fresh = false, deep = false, resume = false;
  u32 em = 0;     // arrivals computed for the current element
  u32 fin = 0;    // slots this warp must finalise (warp-uniform)
  u32 stamp = 0;  // dense-array stamp of this warp
  // lane steps per scheduling round, from the batch's expected arrivals per
  // element at the first pass, k (ln k + 2.5) / (elements per vector): light
  // elements (config 1: ~0.2) are turned over every 2 steps, deep ones (config 2:
  // ~10) walk 6 steps between the warp-level checks
  int u_run;
  {
    const float n_avg = one_vec ? (float)(offsets[1] - offsets[0])
                                : (float)(offsets[n_vec] - offsets[0]) / (float)n_vec;
    const float depth = (float)k * (__logf((float)k) + 2.5f) / fmaxf(n_avg, 1.0f);
    u_run = depth < 2.0f ? GM_URUN0 : depth < 6.0f ? GM_URUN1 : GM_URUN2;
  }
  // the lane's next element, taken and loading while the current one is walked
  bool nx_ok = false;
  int nx_slot = 0;
  u64 nx_id = 0;
  double nx_w = 0.0;
  // WQ: the warp's ticket batch in flight (warp-uniform): slot, element count
  int b_slot = -1;
  u32 b_cnt = 0, b_pos = 0;  // staged elements, elements tested so far
  // elements this lane finished in the current round, per slot (C::FW bits
  // each: at most u_run + 1 per round), and their arrivals (counted mode); the warp adds them up per slot
  // at the end of the round
  u32 dpack = 0;
  u32 emacc[V];
#pragma unroll
  for (int s = 0; s < V; ++s) emacc[s] = 0;

  // count `c` finished elements of slot s (lane 0; the warp's register
  // updates are fenced first).  n is read before the increment: once they are
  // counted the slot may be finalised and reloaded by another warp.
  auto complete_batch = [&](int s, int c, unsigned long long em_sum) {
    __threadfence_block();
    __syncwarp();
    if (lane == 0) {
      SlotInfo& sl = S.slot[s];
      const int n = *(volatile int*)&sl.n;
      if (kCount) atomicAdd(&sl.emitted, em_sum);
      __threadfence_block();
      const int old = atomicAdd(&sl.done, c);
      if (old + c == n) fin |= 1u << s;
    }
    fin = __shfl_sync(FULL, fin, 0);
  };

  // lane-level: take a ticket from the oldest slot with untaken elements and
  // start loading that element (its id and weight are read at start_next)
  auto take_next = [&]() {
    if constexpr (C::WQ > 0) {  // pop a tested survivor from the warp's queue
      const int h = atomicAdd(&q_pos[0], 1);
      if (h >= *(volatile int*)&q_pos[1]) return;  // empty (the refill clamps qhead back)
      const int e = h % C::QCAP;
      nx_id = q_id[e];
      nx_w = q_w[e];
      nx_slot = q_slot[e];
      nx_ok = true;
      return;
    }
    // the slot the CTA is currently handing out (a hint: one 8-byte load
    // instead of the scan over all the slots; rescanned -- oldest slot with
    // untaken elements first -- when it has run dry)
    int best = *(volatile int*)&S.cur;
    {
      const unsigned long long gh = *(volatile unsigned long long*)&S.slot[best].grab;  // (grab, hdr)
      if (!ticket_valid((unsigned)gh, (unsigned)(gh >> 32))) {
        best = -1;
        unsigned bseq = 0xFFFFFFFFu;
#pragma unroll
        for (int s = 0; s < V; ++s) {
          const unsigned long long gh2 = *(volatile unsigned long long*)&S.slot[s].grab;
          const unsigned q = *(volatile unsigned*)&S.slot[s].seq;
          if (ticket_valid((unsigned)gh2, (unsigned)(gh2 >> 32)) && q < bseq) {
            bseq = q;
            best = s;
          }
        }
        if (best < 0) return;
        *(volatile int*)&S.cur = best;
      }
    }
    const unsigned t = atomicAdd(&S.slot[best].grab, 1u);
    __threadfence_block();
    if (!ticket_valid(t, *(volatile unsigned*)&S.slot[best].hdr)) return;  // ran dry meanwhile
    const long long lo = *(volatile long long*)&S.slot[best].lo;
    const u32 i = t & 0xFFFFFFu;
    nx_id = (u64)__ldcg(&ids[lo + i]);  // L2-only loads: each element is read once
    nx_w = (double)__ldcg(&wts[lo + i]);
    nx_slot = best;
    nx_ok = true;
  };
  // lane-level: make the prefetched element the lane's current one
  auto start_next = [&]() {
    SlotInfo& sl = S.slot[nx_slot];
    L.slot = nx_slot;
    L.id = nx_id;
    L.w = nx_w;
    L.tau = sl.tau;
    L.fast = sl.fast != 0;
    L.regs = slot_regs<C>(smem_raw, nx_slot, k);
    L.ubase = sl.useed + nx_id * K_ELEM;
    L.pbase = sl.pseed + nx_id * K_ELEM;
    L.b = 0.0;
    L.z = 0;
    L.used = 0;
    em = 0;
    nx_ok = false;
    if (nx_w >= sl.deep_w) {
      deep = true;
    } else {
      if constexpr (C::LOGM)
        bm_clear<C>(mytab);
      else
        tab_next_element<C>(mytab, L.g24);
      live = true;
      fresh = true;
    }
  };
  // lane-level: note the lane's finished element (counted by the warp at the
  // end of the round)
  auto finish_element = [&]() {
    dpack += 1u << (C::FW * L.slot);
    if constexpr (kCount) {
#pragma unroll
      for (int s = 0; s < V; ++s) emacc[s] += L.slot == s ? em : 0u;
    }
  };

  // count the finished elements per slot (their register updates fenced
  // first); the warp whose count completes a slot finalises it.  Every path
  // through the loop ends with it, so no count stays pending while a warp idles.
  auto flush_counts = [&]() {
    if (u32 any = __reduce_or_sync(FULL, dpack)) {
      __threadfence_block();
      constexpr u32 FM = (1u << C::FW) - 1u;
      // over the slots with finished elements only (one copy of the body:
      // kernel code size)
      for (u32 live_s = 0, am = any; am; am >>= C::FW, ++live_s) {
        if (!(am & FM)) continue;  // no element of slot live_s finished
        const int s = (int)live_s;
        const u32 c = __reduce_add_sync(FULL, (dpack >> (C::FW * s)) & FM);
        u32 em_s = 0;
        if constexpr (kCount) {
#pragma unroll
          for (int s2 = 0; s2 < V; ++s2)
            if (s2 == s) {
              em_s = emacc[s2];
              emacc[s2] = 0;
            }
        }
        const u32 es = kCount ? __reduce_add_sync(FULL, em_s) : 0u;
        if (lane == 0) {
          SlotInfo& sl = S.slot[s];
          const int n = *(volatile int*)&sl.n;  // read before the count: the slot may then be reloaded
          if (kCount) atomicAdd(&sl.emitted, (unsigned long long)es);
          __threadfence_block();
          if (atomicAdd(&sl.done, (int)c) + (int)c == n) fin |= 1u << s;
        }
      }
      fin = __shfl_sync(FULL, fin, 0);
      dpack = 0;
    }
  };

  // WQ (warp-uniform): test the staged batch -- survivors to the queue,
  // elements whose first arrival cannot reach tau counted as finished -- then
  // take the next batch of tickets and start its copies into the staging area
  auto refill = [&]() {
    if (b_slot >= 0) {
      if (b_pos == 0) {
        asm volatile("cp.async.wait_all;\n" ::: "memory");
        __syncwarp();
      }
      SlotInfo& sl = S.slot[b_slot];
      const double tk = *(volatile double*)&sl.tau * (double)k;
      const float tkf = (float)tk;
      const u64 c0 = *(volatile u64*)&sl.useed + K_STEP;
      const int t0 = *(volatile int*)&q_pos[1];
      const int head = min(*(volatile int*)&q_pos[0], t0);  // pops may have run past the tail
      int tail = t0;
      u32 skips = 0;
      for (; b_pos < b_cnt && tail - head + 32 <= C::QCAP; b_pos += 32) {
        const u32 i = b_pos + lane;
        const bool valid = i < b_cnt;
        const u64 id = valid ? (u64)st_id[i] : 0ull;
        const WT wv = valid ? st_w[i] : WT(0);
        const bool sk = valid && filter_skip_f(c0 + id * K_ELEM, filter_x(wv, tkf, tk));
        const bool kp = valid && !sk;
        const unsigned m = __ballot_sync(FULL, kp);
        if (kp) {
          const int e = (tail + __popc(m & lt_mask)) % C::QCAP;
          q_id[e] = id;
          q_w[e] = (double)wv;
          q_slot[e] = b_slot;
        }
        tail += __popc(m);
        skips += sk ? 1u : 0u;
      }
      dpack += skips << (C::FW * b_slot);
      if constexpr (kCount) {
#pragma unroll
        for (int s2 = 0; s2 < V; ++s2) emacc[s2] += b_slot == s2 ? skips : 0u;
      }
      __syncwarp();
      if (lane == 0) {
        q_pos[0] = head;
        __threadfence_block();
        *(volatile int*)&q_pos[1] = tail;
      }
      __syncwarp();
      if (b_pos < b_cnt) return;  // ring full: the rest of the batch waits
      b_slot = -1;
    }
    // the next batch of tickets
    int best = -1;
    u32 base = 0, cnt = 0;
    if (lane == 0) {
      unsigned bseq = 0xFFFFFFFFu;
#pragma unroll
      for (int s2 = 0; s2 < V; ++s2) {
        const unsigned g = *(volatile unsigned*)&S.slot[s2].grab;
        const unsigned h = *(volatile unsigned*)&S.slot[s2].hdr;
        const unsigned q = *(volatile unsigned*)&S.slot[s2].seq;
        if (ticket_valid(g, h) && q < bseq) {
          bseq = q;
          best = s2;
        }
      }
      if (best >= 0) {
        const unsigned t = atomicAdd(&S.slot[best].grab, (unsigned)C::WQ);
        __threadfence_block();
        const unsigned h = *(volatile unsigned*)&S.slot[best].hdr;
        if (ticket_valid(t, h)) {
          base = t & 0xFFFFFFu;
          cnt = min((u32)C::WQ, (h & 0xFFFFFFu) - base);
        } else {
          best = -1;
        }
      }
    }
    best = __shfl_sync(FULL, best, 0);
    if (best < 0) return;
    base = __shfl_sync(FULL, base, 0);
    cnt = __shfl_sync(FULL, cnt, 0);
    const long long lo = *(volatile long long*)&S.slot[best].lo;
    for (u32 i = lane; i < cnt; i += 32) {
      const u32 ds = (u32)__cvta_generic_to_shared(&st_id[i]);
      const u32 dw = (u32)__cvta_generic_to_shared(&st_w[i]);
      if (sizeof(IdT) == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(ds), "l"(&ids[lo + base + i]) : "memory");
      else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(ds), "l"(&ids[lo + base + i]) : "memory");
      if (sizeof(WT) == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dw), "l"(&wts[lo + base + i]) : "memory");
      else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(dw), "l"(&wts[lo + base + i]) : "memory");
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    b_slot = best;
    b_cnt = cnt;
    b_pos = 0;
  };

#ifdef GM_STATS
  long long t_prev = 0;
  int t_sec = 15;
#endif
  for (;;) {
#ifdef GM_STATS
    { const long long now = clock64(); if (lane == 0 && t_prev) atomicAdd(&g_stats[t_sec], (unsigned long long)(now - t_prev)); t_prev = now; t_sec = 8; }
#endif
    // ---- (1) finalise slots whose last elements this warp counted
    while (fin) {
      const int s = __ffs(fin) - 1;
      fin &= fin - 1;
      SlotInfo& sl = S.slot[s];
      __threadfence_block();
      Reg* regs = slot_regs<C>(smem_raw, s, k);
      bool unset = false;
      for (u32 j = lane; j < k; j += 32) unset |= regs[j].y == INF_BITS;
      const int att = __shfl_sync(FULL, *(volatile int*)&sl.attempt, 0);
      if (__any_sync(FULL, unset) && att < 3) {
        if (lane == 0) {
          slot_open_pass(sl, k, att + 1, C::kDeep);
          GM_TRACE((unsigned long long)(sl.v & 0xFFFFFFFF) | ((unsigned long long)(att + 1) << 32) | (2ull << 40) |
                   ((unsigned long long)blockIdx.x << 48) | ((unsigned long long)s << 60));
        }
        __syncwarp();
        continue;
      }
      const int64_t v = __shfl_sync(FULL, *(volatile long long*)&sl.v, 0);
      for (u32 j = lane; j < k; j += 32) {
        const Reg rg = regs[j];
        y_out[v * (int64_t)k + j] = __longlong_as_double((long long)rg.y);
        s_out[v * (int64_t)k + j] = rg.id;
      }
      if (kCount && lane == 0) emitted_out[v] = (int64_t)sl.emitted;
      if (lane == 0)
        GM_TRACE((unsigned long long)(v & 0xFFFFFFFF) | ((unsigned long long)att << 32) | (1ull << 40) |
                 ((unsigned long long)blockIdx.x << 48) | ((unsigned long long)s << 60));
      __syncwarp();
#ifdef GM_STATS
      const long long t_l0 = clock64();
#endif
      slot_load<C, WT>(S, s, smem_raw, k, offsets, n_vec, Wsum, vflags, vec_counter, err, attempt0, lane, vec_list,
                       wts, useed, salt, vseeds, one_vec);
#ifdef GM_STATS
      if (lane == 0) atomicAdd(&g_stats[11], (unsigned long long)(clock64() - t_l0));
#endif
    }

#ifdef GM_STATS
    { const long long now = clock64(); if (lane == 0 && t_prev) atomicAdd(&g_stats[t_sec], (unsigned long long)(now - t_prev)); t_prev = now; t_sec = 9; }
#endif
    // ---- (2) warp walks: deep elements and resumed (table-full) elements
    unsigned dm = __ballot_sync(FULL, deep);
    while (dm) {
      const int src = __ffs(dm) - 1;
      dm &= dm - 1;
      const int s = __shfl_sync(FULL, L.slot, src);
      const u64 wid = __shfl_sync(FULL, L.id, src);
      const double ww = __shfl_sync(FULL, L.w, src);
      const double tau = __shfl_sync(FULL, L.tau, src);
      const bool wres = __shfl_sync(FULL, (int)resume, src) != 0;
      const u32 z0 = wres ? __shfl_sync(FULL, L.z, src) : 0u;
      const double b0 = wres ? __shfl_sync(FULL, L.b, src) : 0.0;
      const bool wfast = __shfl_sync(FULL, (int)L.fast, src) != 0;
      const u32 em0 = kCount ? __shfl_sync(FULL, em, src) : 0u;
      const u64 wus = *(volatile u64*)&S.slot[s].useed, wps = *(volatile u64*)&S.slot[s].pseed;
      if (++stamp > 0xFFFFu) {
        for (u32 i = lane; i < k; i += 32) dense[i] = 0;
        __syncwarp();
        stamp = 1;
      }
      if (C::LOGM && wres) {  // the source lane's drawn positions, traced to their values -> dense array
        const u32* slog = tables + (size_t)NT * (C::BMB * 4) + (warp * 32 + src);
        for (u32 i = lane; i < z0; i += 32) {
          const u32 pos = (slog[(i >> 1) * NT] >> ((i & 1u) * 16)) & 0xFFFFu;
          GM_CHECK(pos < k && z0 <= (u32)C::LOGCAP, 32u);
          if (pos >= z0) dense[pos] = (stamp << 16) | log_trace<C>(slog, pos, z0);
        }
        __syncwarp();
      } else if (wres) {  // the source lane's live table entries -> dense array
        const u32* stab = tables + (warp * 32 + src) * 4;
        const u32 sg24 = __shfl_sync(FULL, L.g24, src);
        for (u32 wi = lane; wi < (u32)C::SLOTS; wi += 32) {
          const u32 e = stab[(wi >> 2) * (NT * 4) + (wi & 3)];
          const u32 pos = (e >> C::PB) & C::VMASK;
          if (tab_live<C>(e, sg24) && pos >= z0) dense[pos] = (stamp << 16) | (e & C::VMASK);
        }
        __syncwarp();
      }
      u32 wem = 0;
      Reg* regs = slot_regs<C>(smem_raw, s, k);
#ifdef GM_WALK_NOINLINE
      csr_walk(wid, ww, tau, k, wus, wps, DenseFlat{dense}, stamp, scan, prov, regs, wem, z0, b0, mtab,
               (u32)C::MTAB, wfast);
#else
      walk_warp<true>(wid, ww, tau, k, wus, wps, dense, stamp, scan, prov, regs, nullptr, wem, z0, b0, mtab,
                      (u32)C::MTAB, ltab, wfast);
#endif
      wem = __shfl_sync(FULL, wem, 0);
      GM_STAT(3, lane == 0);  // warp walks
      GM_STAT(4, lane == 0 ? wem : 0u);
      complete_batch(s, 1, (unsigned long long)(em0 + wem));
      if (lane == src) {
        deep = false;
        resume = false;
      }
    }

#ifdef GM_STATS
    { const long long now = clock64(); if (lane == 0 && t_prev) atomicAdd(&g_stats[t_sec], (unsigned long long)(now - t_prev)); t_prev = now; t_sec = 10; }
#endif
    // ---- (3) lanes without an element start the one they prefetched (or take
    // one now), and every lane keeps its next element in flight
    if constexpr (C::WQ > 0) refill();
    if (!live && !deep) {
      if (!nx_ok) take_next();
      if (nx_ok) start_next();
    }
    if (live && !nx_ok) take_next();

    // ---- exit / idle
    if (!__any_sync(FULL, live || deep)) {
#ifndef GM_IDLE_FLUSH_ALL
      if constexpr (C::WQ > 0) flush_counts();  // (skips counted by a refill)
#else
      flush_counts();
#endif
#ifndef GM_STATS_WALK
      GM_STAT(0, lane == 0);  // idle iterations
#endif
#ifdef GM_STATS
    { const long long now = clock64(); if (lane == 0 && t_prev) atomicAdd(&g_stats[t_sec], (unsigned long long)(now - t_prev)); t_prev = now; t_sec = 12; }
#endif
      bool queued = false;
      if constexpr (C::WQ > 0)
        queued = b_slot >= 0 || *(volatile int*)&q_pos[1] > *(volatile int*)&q_pos[0];
      if (!__any_sync(FULL, nx_ok) && !queued) {
        bool open = false;
#pragma unroll
        for (int s = 0; s < V; ++s) open |= *(volatile int*)&S.slot[s].state != SLOT_EMPTY;
        if (!__shfl_sync(FULL, (int)open, 0)) break;
        __nanosleep(200);
      }
      continue;
    }

    // ---- drain: no slot has untaken elements and few lanes still walk --
    // hand their elements to the warp walker (all 32 lanes on each)
    if (C::DRAIN_LIVE > 0 && !__any_sync(FULL, nx_ok) && __popc(__ballot_sync(FULL, live)) <= C::DRAIN_LIVE) {
      bool work = false;
      if constexpr (C::WQ > 0)
        work = b_slot >= 0 || *(volatile int*)&q_pos[1] > *(volatile int*)&q_pos[0];
      if (lane == 0) {
#pragma unroll
        for (int s = 0; s < V; ++s)
          work |= ticket_valid(*(volatile unsigned*)&S.slot[s].grab, *(volatile unsigned*)&S.slot[s].hdr);
      }
      if (!__shfl_sync(FULL, (int)work, 0)) {
        if (live) {
          em += L.z;
          live = false;
          deep = true;
          resume = true;
        }
#ifndef GM_IDLE_FLUSH_ALL
        if constexpr (C::WQ > 0) flush_counts();
#else
        flush_counts();
#endif
        continue;
      }
    }

#ifdef GM_STATS
    { const long long now = clock64(); if (lane == 0 && t_prev) atomicAdd(&g_stats[t_sec], (unsigned long long)(now - t_prev)); t_prev = now; t_sec = 13; }
#endif
    // ---- (4) u_run lane steps; a lane whose element ends counts it and goes on
    // with its prefetched element at the next step
#pragma unroll 1
    for (int u = 0; u < u_run; ++u) {
#ifdef GM_STATS
      {
        const unsigned lv = __ballot_sync(FULL, live), dp = __ballot_sync(FULL, deep);
        const unsigned nn = __ballot_sync(FULL, !live && !deep);
        bool avail = false;
#pragma unroll
        for (int s2 = 0; s2 < V; ++s2)
          avail |= ticket_valid(*(volatile unsigned*)&S.slot[s2].grab, *(volatile unsigned*)&S.slot[s2].hdr);
#ifndef GM_STATS_WALK
        if (lane == 0 && !avail) atomicAdd(&g_stats[7], (unsigned long long)__popc(nn));
        if (lane == 0) {
          atomicAdd(&g_stats[1], 1ull);
          atomicAdd(&g_stats[2], (unsigned long long)__popc(lv));
          atomicAdd(&g_stats[5], (unsigned long long)__popc(dp));
          atomicAdd(&g_stats[6], (unsigned long long)__popc(nn));
        }
#endif
      }
#endif
      if (live) {
        int rc;
        if constexpr (C::LOGM)
          rc = lane_step_log<C>(L, fresh, mytab, mylog, mtab64, k, ltab);
        else
          rc = lane_step<C>(L, fresh, mytab, mtab64, k, ltab);
        fresh = false;
        if (rc == 1) {
          if (kCount) em += L.z < k ? L.z + 1 : L.z;
          live = false;
          finish_element();
          if (nx_ok) start_next();
        } else if (rc == 2) {
          if (kCount) em += L.z;
          live = false;
          deep = true;
          resume = true;
        }
      }
    }
#ifdef GM_STATS
    { const long long now = clock64(); if (lane == 0 && t_prev) atomicAdd(&g_stats[t_sec], (unsigned long long)(now - t_prev)); t_prev = now; t_sec = 14; }
#endif
    // ---- (5) count the round's finished elements
    flush_counts();
  }
}

}  // namespace gmk
