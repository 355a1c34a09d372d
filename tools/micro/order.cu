// Does an LDS wait behind an outstanding ATOMS.CAS.128 / ATOMS.MIN.U64 of the same warp?
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2302_05176_b200/csrc/gm_core.cuh"
using namespace gmk;

template <int MODE>
__global__ void k(unsigned long long* cyc, u64* sink, int iters) {
  __shared__ Reg r[1024];
  __shared__ u32 chase[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) { r[i].y = ~0ull >> 1; r[i].id = ~0ull; chase[i] = (i * 7 + 1) & 1023; }
  __syncthreads();
  u32 x = threadIdx.x;
  u64 acc = 0, oy = 0, oid = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (MODE == 1) {  // CAS (result unused until the end) then dependent LDS chase
      cas128_shared(&r[(threadIdx.x * 33 + i * 97) & 1023], r[0].y, r[0].id, (1ull << 60) - i, i, oy, oid);
      acc += oy;
    } else if (MODE == 2) {  // 64-bit atomicMin (result unused) then chase
      atomicMin((unsigned long long*)&r[(threadIdx.x * 33 + i * 97) & 1023].y, (unsigned long long)((1ull << 60) - i));
    }
    x = chase[x];  // dependent LDS chain
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  sink[threadIdx.x] = acc + x + oid;
}

int main() {
  unsigned long long* cyc; u64* sink;
  cudaMalloc(&cyc, 8); cudaMalloc(&sink, 1024 * 8);
  const char* nm[] = {"LDS chase alone", "CAS128 + LDS chase", "atomicMin64 + LDS chase"};
  for (int m = 0; m < 3; ++m) for (int rep = 0; rep < 2; ++rep) {
    if (m == 0) k<0><<<1, 32>>>(cyc, sink, 4000);
    if (m == 1) k<1><<<1, 32>>>(cyc, sink, 4000);
    if (m == 2) k<2><<<1, 32>>>(cyc, sink, 4000);
    cudaDeviceSynchronize();
    unsigned long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    if (rep) printf("%-26s %7.1f cycles/iter\n", nm[m], (double)c / 4000);
  }
  return 0;
}
