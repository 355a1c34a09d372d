// Decompose the lane step latency: variants of the step body on 1 warp/SM.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2302_05176_b200/csrc/gm_csr.cuh"
using namespace gmk;
using C = CsrCfg<256, 16, 2, 2>;

template <int MODE>
__global__ void __launch_bounds__(256) kvar(unsigned long long* cyc, double* sink, int iters, u32 k) {
  extern __shared__ __align__(16) unsigned char sm[];
  Reg* regs = reinterpret_cast<Reg*>(sm);
  u32* tables = reinterpret_cast<u32*>(sm + (size_t)k * 16);
  u32* mtab = tables + 256 * C::SLOTS;
  for (u32 z = threadIdx.x; z < (u32)C::MTAB; z += blockDim.x) mtab[z] = (z >= 1 && z <= k) ? barrett_magic(k - z + 1) : 0u;
  for (u32 j = threadIdx.x; j < k; j += blockDim.x) { regs[j].y = INF_BITS; regs[j].id = NO_ID; }
  u32* mytab = tables + threadIdx.x * 4;
  tab_clear<C>(mytab);
  __syncthreads();
  const u64 ub = 12345 + threadIdx.x * K_ELEM, pb = 777 + threadIdx.x * K_ELEM;
  const double w = 1.3;
  double b = 0.0, acc = 0.0;
  u32 z = 1, accu = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (MODE == 0) {  // spacing only (chained through b)
      b = __dadd_rn(b, spacing_t<true>(ub, z, w, k));
    } else if (MODE == 1) {  // perm draw + 2 probes (chained through z)
      const u64 g = mix64(pb + (u64)z * K_STEP);
      const u32 m = k - z + 1, M = mtab[z];
      u32 r = mod_barrett((u32)(g >> 32), m, M);
      r = mod_barrett((r << 16) | ((u32)g >> 16), m, M);
      r = mod_barrett((r << 16) | ((u32)g & 0xFFFFu), m, M);
      const u32 ji = z - 1 + r;
      const uint4 qz = tab_bucket<C>(mytab, (z - 1) & 15), qj = tab_bucket<C>(mytab, ji & 15);
      accu += probe_min(qz, z - 1) + probe_min(qj, ji);
      z = 1 + (accu & 63);
    } else if (MODE == 2) {  // reg_min chain
      reg_min<true>(&regs[(threadIdx.x * 31 + i * 7) & (k - 1)], (u64)(1ull << 60) - i, (u64)i);
      accu += 1;
    } else if (MODE == 3) {  // spacing + perm/probes independent (ILP) chained via b and z
      const double d = spacing_t<true>(ub, z, w, k);
      const u64 g = mix64(pb + (u64)z * K_STEP);
      const u32 m = k - z + 1, M = mtab[z];
      u32 r = mod_barrett((u32)(g >> 32), m, M);
      r = mod_barrett((r << 16) | ((u32)g >> 16), m, M);
      r = mod_barrett((r << 16) | ((u32)g & 0xFFFFu), m, M);
      const u32 ji = z - 1 + r;
      const uint4 qz = tab_bucket<C>(mytab, (z - 1) & 15), qj = tab_bucket<C>(mytab, ji & 15);
      accu += probe_min(qz, z - 1) + probe_min(qj, ji);
      b = __dadd_rn(b, d);
      z = 1 + (accu & 63);
    } else if (MODE == 4) {  // log_pos only
      acc = -log_pos(acc * 0.25 + 0.3);
    } else if (MODE == 5) {  // ddiv_fast only
      acc = ddiv_fast(acc + 1.0, w * (double)(k - z + 1));
    } else if (MODE == 6) {  // u_open(mix64)
      acc += u_open(mix64(ub + (u64)(acc > 2.0) + i));
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) atomicAdd(cyc, (unsigned long long)(t1 - t0));
  sink[threadIdx.x] = b + acc + accu;
}

template <int MODE>
void run(const char* name, unsigned long long* cyc, double* sink, size_t smem) {
  cudaFuncSetAttribute(kvar<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(cyc, 0, 8);
    kvar<MODE><<<1, 32, smem>>>(cyc, sink, 2000, 1024);
    cudaDeviceSynchronize();
    unsigned long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    if (rep) printf("%-28s %7.1f cycles/iter\n", name, (double)c / 2000);
  }
}

int main() {
  unsigned long long* cyc;
  double* sink;
  cudaMalloc(&cyc, 8);
  cudaMalloc(&sink, 256 * 8);
  const size_t smem = (size_t)1024 * 16 + 256 * C::SLOTS * 4 + C::MTAB * 4;
  run<0>("spacing (b chain)", cyc, sink, smem);
  run<1>("perm+2 probes (z chain)", cyc, sink, smem);
  run<2>("reg_min", cyc, sink, smem);
  run<3>("spacing || perm+probes", cyc, sink, smem);
  run<4>("log_pos", cyc, sink, smem);
  run<5>("ddiv_fast", cyc, sink, smem);
  run<6>("u_open(mix64)", cyc, sink, smem);
  return 0;
}
