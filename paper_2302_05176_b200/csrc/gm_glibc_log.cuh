// gm_glibc_log.cuh -- the host C library's double `log`, bit for bit, on the device.
//
// The reference computes every arrival's spacing with CPython's math.log
// (randgen.py:186), i.e. glibc's log.  glibc 2.39 on x86-64 resolves `log`
// (an ifunc) to its FMA variant on any CPU with FMA + AVX2; that variant is
// the table-driven algorithm of sysdeps/ieee754/dbl-64/e_log.c compiled with
// FMA contraction.  This file restates the operation sequence of that
// compiled function (read from the image's libm.so.6 disassembly, one line
// per instruction below), with every multiply, add and fused multiply-add
// pinned to round-to-nearest so nvcc cannot re-associate or contract them:
// the same inputs give the same bits as the host's log.  Data (ln2 hi/lo, the
// two polynomials, the 128 x {invc, logc} table) come from the same library
// (tools/gen_glibc_log.py -> gm_glibc_logtab.h).  Verified against libm's
// log on the host (tests/test_glibc_log.py, every input class) and on the
// device (tests/test_gpu_parity.py test_device_log_is_glibc_log).
//
// Domain: positive normal doubles (the sketch's uniforms are in
// [2^-54, 1]); glibc's special-case branch (zero, subnormal, negative, inf,
// nan) is not restated.
#pragma once

#include <cstdint>

#include "gm_glibc_logtab.h"

#if defined(__CUDACC__)
#define GM_GLOG_HD __host__ __device__ __forceinline__
#else
#define GM_GLOG_HD inline
#include <cmath>
#include <cstring>
#endif

namespace gmk {

// The polynomial and ln2 constants.  On the device they live in the constant
// bank: the walkers load them with LDCU.128 / LDC.64 (two constants per
// load), where a literal double with a full 64-bit pattern costs two moves
// per use (ptxas re-materialises them in the walkers' loops): 10 fewer
// instructions in the main branch, 12 in the near-1 branch (K1 config 3 1%
// faster, the roofline probe 6%; GM_GLOG_LITERAL restores the literals).
#if defined(__CUDACC__) && !defined(GM_GLOG_LITERAL)
enum { GKI_LN2HI, GKI_LN2LO, GKI_A0, GKI_A1, GKI_A2, GKI_A3, GKI_A4, GKI_B0, GKI_B1, GKI_B2, GKI_B3, GKI_B4, GKI_B5,
       GKI_B6, GKI_B7, GKI_B8, GKI_B9, GKI_B10, GKI_N };
__constant__ double gm_glog_k[GKI_N] = {GM_GLOG_LN2HI, GM_GLOG_LN2LO, GM_GLOG_A0, GM_GLOG_A1, GM_GLOG_A2, GM_GLOG_A3,
                                        GM_GLOG_A4,    GM_GLOG_B0,    GM_GLOG_B1, GM_GLOG_B2, GM_GLOG_B3, GM_GLOG_B4,
                                        GM_GLOG_B5,    GM_GLOG_B6,    GM_GLOG_B7, GM_GLOG_B8, GM_GLOG_B9, GM_GLOG_B10};
#endif
#if defined(__CUDA_ARCH__) && !defined(GM_GLOG_LITERAL)
#define GK(n) gm_glog_k[GKI_##n]
#else
#define GK(n) GM_GLOG_##n
#endif

#if defined(__CUDA_ARCH__)
#define GLF(a, b, c) __fma_rn((a), (b), (c))
#define GLM(a, b) __dmul_rn((a), (b))
#define GLA(a, b) __dadd_rn((a), (b))
#define GLS(a, b) __dsub_rn((a), (b))
#else
#define GLF(a, b, c) std::fma((a), (b), (c))
#define GLM(a, b) ((a) * (b))  // host builds use -ffp-contract=off
#define GLA(a, b) ((a) + (b))
#define GLS(a, b) ((a) - (b))
#endif

GM_GLOG_HD uint64_t glog_bits(double x) {
#if defined(__CUDA_ARCH__)
  return (uint64_t)__double_as_longlong(x);
#else
  uint64_t u;
  std::memcpy(&u, &x, 8);
  return u;
#endif
}

GM_GLOG_HD double glog_from_bits(uint64_t u) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double((long long)u);
#else
  double x;
  std::memcpy(&x, &u, 8);
  return x;
#endif
}

// Near-1 branch: 1 - 2^-4 <= x < 1 + 0x1.09p-4 (x != 1).  Degree-11 polynomial
// in r = x - 1 with the leading r - r^2/2 split exactly (rhi: r rounded to 26
// bits via r + r 2^27 - r 2^27).
GM_GLOG_HD double glibc_log_near1(double x) {
  const double r = GLS(x, 1.0);                         // vsubsd 1.0
  double p2 = GLF(r, GK(B2), GK(B1));            // vfmadd213sd B1
  double p3 = GLF(r, GK(B5), GK(B4));            // vfmadd213sd B4
  const double r2 = GLM(r, r);                           // vmulsd
  double p5 = GLF(r, GK(B8), GK(B7));            // vfmadd213sd B7
  p2 = GLF(r2, GK(B3), p2);                          // vfmadd231sd B3
  p3 = GLF(r2, GK(B6), p3);                          // vfmadd231sd B6
  const double r3 = GLM(r, r2);                          // vmulsd
  double q = GLF(r2, GK(B9), p5);                    // vfmadd132sd B9
  q = GLF(r3, GK(B10), q);                           // vfmadd231sd B10
  q = GLF(q, r3, p3);                                    // vfmadd132sd
  q = GLF(q, r3, p2);                                    // vfmadd132sd
  const double t = GLF(r, 0x1p27, r);                    // r + w, w = r 2^27 (exact product)
  const double rhi = GLF(-0x1p27, r, t);                 // vfnmadd132sd: (r + w) - w
  const double rhi2 = GLM(rhi, rhi);                     // vmulsd
  const double rlo = GLS(r, rhi);                        // vsubsd
  const double hi = GLF(rhi2, GM_GLOG_B0, r);            // vfmadd132sd: r + rhi^2 B0
  const double d = GLS(r, hi);                           // vsubsd
  const double rs = GLA(r, rhi);                         // vaddsd
  double lo = GLF(rhi2, GM_GLOG_B0, d);                  // vfmadd132sd: r - hi + rhi^2 B0
  lo = GLF(GLM(GM_GLOG_B0, rlo), rs, lo);                // vmulsd; vfmadd132sd
  const double y = GLF(q, r3, lo);                       // vfmadd132sd
  return GLA(hi, y);                                     // vaddsd
}

// Main branch: x = 2^k z, z in [0x1.6p-1, 0x1.6p0), i from the top 7 bits of
// z's mantissa; log x = k ln2 + logc + log1p(r), r = z invc - 1 (one fma).
// tab: 128 x {invc, logc} (global or shared memory, 16-byte aligned rows).
template <class TabT>
GM_GLOG_HD double glibc_log_main(double x, const TabT* tab) {
  const uint64_t ix = glog_bits(x);
  const uint64_t tmp = ix - 0x3fe6000000000000ull;
  const uint32_t i = (uint32_t)(tmp >> 45) & 127u;
  const int k = (int)((int64_t)tmp >> 52);
  const double z = glog_from_bits(ix - (tmp & 0xfff0000000000000ull));
  const double kd = (double)k;                           // vcvtsi2sd (32-bit)
#if defined(__CUDA_ARCH__)
  const double2 c = *reinterpret_cast<const double2*>(&tab[2 * i]);
  const double invc = c.x, logc = c.y;
#else
  const double invc = tab[2 * i], logc = tab[2 * i + 1];
#endif
  const double w = GLF(kd, GK(LN2HI), logc);         // vfmadd213sd logc
  const double r = GLF(z, invc, -1.0);                   // vfmadd132sd invc, -1
  const double a21 = GLF(r, GK(A2), GK(A1));     // vfmadd213sd A1
  const double hi = GLA(r, w);                           // vaddsd
  const double r2 = GLM(r, r);                           // vmulsd
  double lo = GLA(GLS(w, hi), r);                        // vsubsd; vaddsd
  lo = GLF(kd, GK(LN2LO), lo);                       // vfmadd231sd ln2lo
  const double rr2 = GLM(r, r2);                         // vmulsd
  const double a43 = GLF(r, GK(A4), GK(A3));     // vfmadd132sd A4
  lo = GLF(r2, GK(A0), lo);                          // vfmadd231sd A0
  const double p = GLF(a43, r2, a21);                    // vfmadd132sd
  const double y = GLF(rr2, p, lo);                      // vfmadd132sd
  return GLA(y, hi);                                     // vaddsd
}

GM_GLOG_HD bool glibc_log_is_near1(double x) {
  return glog_bits(x) - 0x3fee000000000000ull < 0x3090000000000ull;
}

// log(x) for a positive normal double x, equal to the host libm's log.
template <class TabT>
GM_GLOG_HD double glibc_log_t(double x, const TabT* tab) {
  const uint64_t ix = glog_bits(x);
  if (glibc_log_is_near1(x)) return ix == 0x3ff0000000000000ull ? 0.0 : glibc_log_near1(x);
  return glibc_log_main(x, tab);
}

#undef GLF
#undef GLM
#undef GLA
#undef GLS
#undef GK

}  // namespace gmk
