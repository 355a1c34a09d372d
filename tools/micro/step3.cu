#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2302_05176_b200/csrc/gm_csr.cuh"
using namespace gmk;
using C = CsrCfg<256, 16, 2, 2>;
namespace gmk {
#include "lane_step_t.inc"
}
__global__ void __launch_bounds__(256) kstep(unsigned long long* acc, int iters, u32 k) {
  extern __shared__ __align__(16) unsigned char sm[];
  Reg* regs = reinterpret_cast<Reg*>(sm);
  u32* tables = reinterpret_cast<u32*>(sm + (size_t)k * 16);
  u32* mtab = tables + 256 * C::SLOTS;
  for (u32 z = threadIdx.x; z < (u32)C::MTAB; z += blockDim.x) mtab[z] = (z >= 1 && z <= k) ? barrett_magic(k - z + 1) : 0u;
  for (u32 j = threadIdx.x; j < k; j += blockDim.x) { regs[j].y = INF_BITS; regs[j].id = NO_ID; }
  u32* mytab = tables + threadIdx.x * 4;
  tab_clear<C>(mytab);
  __syncthreads();
  Lane L;
  L.regs = regs; L.fast = true; L.tau = 9.43 / 1000.0;
  u64 e = threadIdx.x * 977;
  bool fresh = true;
  auto start = [&]() {
    e += 7919;
    L.id = e; L.w = 1.0 + (double)((e * 2654435761u) % 1000) / 500.0; L.ubase = 1 + L.id * K_ELEM; L.pbase = 2 + L.id * K_ELEM;
    L.b = 0; L.z = 0; L.used = 0; tab_clear<C>(mytab); fresh = true;
  };
  start();
  long long T[7];
  unsigned long long sum[7] = {0};
  long long tl = clock64();
  for (int i = 0; i < iters; ++i) {
    const int rc = lane_step_t<C>(L, fresh, mytab, mtab, k, T);
    const long long te = clock64();
    sum[0] += T[0] - tl;
    for (int q = 1; q < 7; ++q) sum[q] += T[q] - T[q - 1];
    tl = te;
    fresh = false;
    if (rc) start();
  }
  if (threadIdx.x == 0) for (int q = 0; q < 7; ++q) acc[q] = sum[q];
}
int main() {
  unsigned long long* acc; cudaMalloc(&acc, 7 * 8);
  const u32 k = 1024;
  const size_t smem = (size_t)k * 16 + 256 * C::SLOTS * 4 + C::MTAB * 4;
  cudaFuncSetAttribute(kstep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int rep = 0; rep < 2; ++rep) { kstep<<<1, 32, smem>>>(acc, 2000, k); cudaDeviceSynchronize(); }
  unsigned long long h[7]; cudaMemcpy(h, acc, 56, cudaMemcpyDeviceToHost);
  const char* nm[] = {"loop/start+branch", "perm draw", "probes issue", "spacing issue", "slow-check", "table+CAS", "t=b+dq"};
  for (int q = 0; q < 7; ++q) printf("%-18s %7.1f cycles/step\n", nm[q], (double)h[q] / 2000);
  return 0;
}
