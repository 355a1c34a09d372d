// Shared-memory atomic throughput (1 CTA of 1024 threads per SM, whole GPU).
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2302_05176_b200/csrc/gm_core.cuh"
using namespace gmk;

template <int MODE>
__global__ void __launch_bounds__(1024) k(unsigned long long* out, int n) {
  __shared__ Reg r[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) { r[i].y = ~0ull >> 1; r[i].id = ~0ull; }
  __syncthreads();
  u64 acc = 0;
  u64 v = (1ull << 62) + threadIdx.x;
  for (int i = 0; i < n; ++i) {
    Reg* p = &r[(threadIdx.x * 37 + i * 101) & 2047];
    if (MODE == 0) {  // 128-bit CAS, result used next iteration
      u64 oy, oid;
      cas128_shared(p, p->y, p->id, v - i, (u64)i, oy, oid);
      acc += oy;
    } else if (MODE == 1) {  // 64-bit atomicMin
      acc += atomicMin((unsigned long long*)&p->y, (unsigned long long)(v - i));
    } else if (MODE == 2) {  // 64-bit atomicMin, result unused
      atomicMin((unsigned long long*)&p->y, (unsigned long long)(v - i));
    } else if (MODE == 3) {  // 64-bit CAS
      acc += atomicCAS((unsigned long long*)&p->y, p->y, (unsigned long long)(v - i));
    } else {  // plain LDS.128 + STS (no atomic)
      const Reg q = *p;
      acc += q.y;
      p->id = (u64)i;
    }
  }
  if (acc == 12345) out[0] = acc;
}

int main() {
  unsigned long long* out;
  cudaMalloc(&out, 8);
  const int n = 2048, blocks = 148;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char* names[] = {"cas128", "min64 (ret)", "min64 (noret)", "cas64", "lds128+sts"};
  for (int m = 0; m < 5; ++m) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      switch (m) {
        case 0: k<0><<<blocks, 1024>>>(out, n); break;
        case 1: k<1><<<blocks, 1024>>>(out, n); break;
        case 2: k<2><<<blocks, 1024>>>(out, n); break;
        case 3: k<3><<<blocks, 1024>>>(out, n); break;
        default: k<4><<<blocks, 1024>>>(out, n); break;
      }
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double ops = (double)blocks * 1024 * n;
      if (rep) printf("%-14s %8.2f Gop/s  %6.2f thread-ops/clk/SM (1.9 GHz)\n", names[m], ops / ms / 1e6, ops / (ms * 1e-3) / 148 / 1.9e9);
    }
  }
  return 0;
}
