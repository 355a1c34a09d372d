// Cycles per lane step of the real lane_step (gm_csr.cuh) on synthetic
// elements: W warps per CTA, one CTA per SM.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2302_05176_b200/csrc/gm_csr.cuh"
using namespace gmk;
using C = CsrCfg<256, 16, 2, 2>;

__global__ void __launch_bounds__(256, 2) kstep(unsigned long long* cyc, unsigned long long* steps_out, int iters, u32 k) {
  extern __shared__ __align__(16) unsigned char sm[];
  Reg* regs = reinterpret_cast<Reg*>(sm);
  u32* tables = reinterpret_cast<u32*>(sm + (size_t)k * 16);
  u32* mtab = tables + 256 * C::SLOTS;
  double (*ltab)[4] = reinterpret_cast<double (*)[4]>(mtab + C::MTAB);
  for (u32 i = threadIdx.x; i < 512; i += blockDim.x) ltab[i >> 2][i & 3] = gm_logtab[i >> 2][i & 3];
  for (u32 z = threadIdx.x; z < (u32)C::MTAB; z += blockDim.x) mtab[z] = (z >= 1 && z <= k) ? barrett_magic(k - z + 1) : 0u;
  for (u32 j = threadIdx.x; j < k; j += blockDim.x) { regs[j].y = INF_BITS; regs[j].id = NO_ID; }
  u32* mytab = tables + threadIdx.x * 4;
  tab_clear<C>(mytab);
  __syncthreads();
  Lane L;
  L.regs = regs; L.fast = true; L.tau = 9.43 / 1000.0;
  u64 e = (u64)blockIdx.x * 100000 + threadIdx.x * 977;
  bool fresh = true;
  auto start = [&]() {
    e += 7919;
    L.id = e; L.w = 1.0 + (double)((e * 2654435761u) % 1000) / 500.0; L.ubase = 1 + L.id * K_ELEM; L.pbase = 2 + L.id * K_ELEM;
    L.b = 0; L.z = 0; L.used = 0; tab_clear<C>(mytab); fresh = true;
  };
  start();
  unsigned long long nsteps = 0;
  __syncwarp();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#ifdef LA
    u32 em = 0;
    const int rc = lane_step_la<C, 4>(L, mytab, mtab, k, ltab, em);
    nsteps += 4;
#else
    const int rc = lane_step<C>(L, fresh, mytab, mtab, k, ltab);
    ++nsteps;
#endif
    fresh = false;
    if (rc) start();
  }
  long long t1 = clock64();
  if ((threadIdx.x & 31) == 0) { atomicAdd(cyc, (unsigned long long)(t1 - t0)); atomicAdd(steps_out, (unsigned long long)nsteps); }
}

int main() {
  unsigned long long *cyc, *st;
  cudaMalloc(&cyc, 8); cudaMalloc(&st, 8);
  const u32 k = 1024;
  const size_t smem = (size_t)k * 16 + 256 * C::SLOTS * 4 + C::MTAB * 4 + 4096;
  cudaFuncSetAttribute(kstep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int warps : {1, 2, 4, 8}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(cyc, 0, 8); cudaMemset(st, 0, 8);
      kstep<<<148, warps * 32, smem>>>(cyc, st, 2000, k);
      cudaDeviceSynchronize();
      unsigned long long c, s;
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost); cudaMemcpy(&s, st, 8, cudaMemcpyDeviceToHost);
      if (rep) printf("warps/SM %2d: %7.1f cycles per warp-step (%s)\n", warps, (double)c / s, cudaGetErrorString(cudaGetLastError()));
    }
  }
  for (int ctas : {2}) for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(cyc, 0, 8); cudaMemset(st, 0, 8);
    kstep<<<148 * ctas, 256, smem>>>(cyc, st, 2000, k);
    cudaDeviceSynchronize();
    unsigned long long c, s;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost); cudaMemcpy(&s, st, 8, cudaMemcpyDeviceToHost);
    if (rep) printf("warps/SM %d: %7.1f cycles per warp-step, %.3f steps/cycle/SM\n", 8 * ctas, (double)c / s, 8.0 * ctas * 32 / ((double)c / s));
  }
  return 0;
}
