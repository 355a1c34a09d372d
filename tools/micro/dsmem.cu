// Latency of 128-bit CAS on shared memory: ATOMS (shared::cta), generic ATOM on
// a local shared address, and shared::cluster on the peer CTA of a 2-CTA
// cluster (distributed shared memory).  One warp, dependent chain.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dsmem tools/micro/dsmem.cu && ./dsmem
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
typedef unsigned long long u64;

__device__ __forceinline__ void cas_cta(unsigned a, u64 cy, u64 cid, u64 ny, u64 nid, u64& oy, u64& oid) {
  asm volatile("{\n\t.reg .b128 d, b, c;\n\tmov.b128 b, {%3, %4};\n\tmov.b128 c, {%5, %6};\n\t"
               "atom.relaxed.cta.shared::cta.cas.b128 d, [%2], b, c;\n\tmov.b128 {%0, %1}, d;\n\t}"
               : "=l"(oy), "=l"(oid) : "r"(a), "l"(cy), "l"(cid), "l"(ny), "l"(nid) : "memory");
}
__device__ __forceinline__ void cas_gen(const void* p, u64 cy, u64 cid, u64 ny, u64 nid, u64& oy, u64& oid) {
  asm volatile("{\n\t.reg .b128 d, b, c;\n\tmov.b128 b, {%3, %4};\n\tmov.b128 c, {%5, %6};\n\t"
               "atom.relaxed.cluster.cas.b128 d, [%2], b, c;\n\tmov.b128 {%0, %1}, d;\n\t}"
               : "=l"(oy), "=l"(oid) : "l"(p), "l"(cy), "l"(cid), "l"(ny), "l"(nid) : "memory");
}
__device__ __forceinline__ void cas_clu(unsigned a, u64 cy, u64 cid, u64 ny, u64 nid, u64& oy, u64& oid) {
  asm volatile("{\n\t.reg .b128 d, b, c;\n\tmov.b128 b, {%3, %4};\n\tmov.b128 c, {%5, %6};\n\t"
               "atom.relaxed.cluster.shared::cluster.cas.b128 d, [%2], b, c;\n\tmov.b128 {%0, %1}, d;\n\t}"
               : "=l"(oy), "=l"(oid) : "r"(a), "l"(cy), "l"(cid), "l"(ny), "l"(nid) : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) bench(long long* out, int iters) {
  __shared__ __align__(16) u64 reg[64][2];
  cg::cluster_group cl = cg::this_cluster();
  const int lane = threadIdx.x;
  reg[lane][0] = 0;
  reg[lane][1] = 0;
  cl.sync();
  if (cl.block_rank() == 0) {
    u64 y = 0, id = 0;
    const unsigned la = (unsigned)__cvta_generic_to_shared(&reg[lane][0]);
    unsigned ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 1;" : "=r"(ra) : "r"(la));
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) { u64 oy, oid; cas_cta(la, y, id, y + 1, id, oy, oid); y = oy + 1; id = oid; }
    long long t1 = clock64();
    for (int i = 0; i < iters; ++i) { u64 oy, oid; cas_gen(&reg[lane][0], y, id, y + 1, id, oy, oid); y = oy + 1; id = oid; }
    long long t2 = clock64();
    y = 0; id = 0;
    for (int i = 0; i < iters; ++i) { u64 oy, oid; cas_clu(ra, y, id, y + 1, id, oy, oid); y = oy + 1; id = oid; }
    long long t3 = clock64();
    if (lane == 0) { out[0] = (t1 - t0) / iters; out[1] = (t2 - t1) / iters; out[2] = (t3 - t2) / iters; out[3] = (long long)y; }
  }
  cl.sync();
}

int main() {
  long long* d;
  cudaMalloc(&d, 8 * sizeof(long long));
  bench<<<2, 32>>>(d, 2000);
  bench<<<2, 32>>>(d, 2000);
  long long h[4];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("cycles per dependent 128-bit CAS (1 warp): shared::cta %lld, generic on local smem %lld, shared::cluster remote %lld (check %lld) err=%s\n",
         h[0], h[1], h[2], h[3], cudaGetErrorString(cudaGetLastError()));
  return 0;
}
