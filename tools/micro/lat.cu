// Latency microbenchmarks (one warp): cycles per dependent operation.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2302_05176_b200/csrc/gm_core.cuh"
using namespace gmk;

__global__ void k_dfma(double* out, long long* cyc, int n, double a) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __fma_rn(x, a, 0.5);
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_mix(u64* out, long long* cyc, int n, u64 a) {
  u64 x = a + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = mix64(x);
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_log(double* out, long long* cyc, int n, double a) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = -log_pos(x) * 0.25 + 0.3;   // stays in (0,1)
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_spacing(double* out, long long* cyc, int n, double w) {
  double b = 0.0; u64 base = 12345 + threadIdx.x * K_ELEM;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { b = __dadd_rn(b, spacing_t<true>(base, 1 + (i & 511), w, 1024)); base += (u64)__double_as_longlong(b) & 1; }
  long long t1 = clock64();
  out[threadIdx.x] = b; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_lds(u32* out, long long* cyc, int n) {
  __shared__ u32 s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (i * 7 + 1) & 1023;
  __syncthreads();
  u32 x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = s[x];
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_cas(u64* out, long long* cyc, int n) {
  __shared__ Reg r[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) { r[i].y = ~0ull >> 1; r[i].id = ~0ull; }
  __syncthreads();
  u64 v = 1ull << 62;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { reg_min<true>(&r[(threadIdx.x * 33 + i * 97) & 1023], v, (u64)i); v -= 1; }
  long long t1 = clock64();
  out[threadIdx.x] = v; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_i2f(double* out, long long* cyc, int n) {
  u64 x = 1234567 + threadIdx.x; double acc = 0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { double d = __ull2double_rn(x); x = (u64)__double_as_longlong(d) >> 3; acc += d; }
  long long t1 = clock64();
  out[threadIdx.x] = acc; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  double* dout; u64* uout; u32* wout; long long* cyc; long long h;
  cudaMalloc(&dout, 1024 * 8); cudaMalloc(&uout, 1024 * 8); cudaMalloc(&wout, 1024 * 4); cudaMalloc(&cyc, 8);
  const int n = 4096;
  auto rep = [&](const char* name, int per) { cudaDeviceSynchronize(); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("%-12s %8.1f cycles/op\n", name, (double)h / n / per); };
  for (int it = 0; it < 2; ++it) {
    k_dfma<<<1, 32>>>(dout, cyc, n, 0.999); rep("dfma", 1);
    k_mix<<<1, 32>>>(uout, cyc, n, 77); rep("mix64", 1);
    k_log<<<1, 32>>>(dout, cyc, n, 0.5); rep("log_pos+2", 1);
    k_spacing<<<1, 32>>>(dout, cyc, n, 1.3); rep("spacing+add", 1);
    k_lds<<<1, 32>>>(wout, cyc, n); rep("lds chase", 1);
    k_cas<<<1, 32>>>(uout, cyc, n); rep("reg_min cas", 1);
    k_i2f<<<1, 32>>>(dout, cyc, n); rep("i2f.f64.u64+", 1);
  }
  return 0;
}
