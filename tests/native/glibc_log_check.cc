// Host check of the device clone of glibc's log (gm_glibc_log.cuh): the
// clone, compiled for the host with every fused multiply-add explicit
// (std::fma) and no contraction, against libm's own log.
//   glibc_log_check N SEED  -> prints "mismatches checked" per input class
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "../../paper_2302_05176_b200/csrc/gm_glibc_log.cuh"

static uint64_t mix64(uint64_t x) {  // randgen.py:64-69
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

int main(int argc, char** argv) {
  const long long n = argc > 1 ? atoll(argv[1]) : 1000000;
  const uint64_t seed = argc > 2 ? strtoull(argv[2], nullptr, 0) : 1;
  const double* tab = &gm_glog_tab[0][0];
  long long bad[4] = {0, 0, 0, 0}, near1 = 0;
  for (long long i = 0; i < n; ++i) {
    const uint64_t h = mix64(seed + (uint64_t)i * 0x9E3779B97F4A7C15ull);
    double xs[4];
    // (0) the sketch's uniforms: (h >> 11) 2^-53 + 2^-54 (randgen.py:119)
    xs[0] = (double)(h >> 11) * 0x1p-53 + 0x1p-54;
    // (1) the near-1 interval [1 - 2^-4, 1 + 0x1.09p-4) and just outside it
    xs[1] = 0.93 + (double)(h >> 11) * 0x1p-53 * 0.14;
    // (2) any positive normal double (random exponent and mantissa)
    const uint64_t e = 1 + (mix64(h) % 2046);
    xs[2] = gmk::glog_from_bits((e << 52) | (h & 0xFFFFFFFFFFFFFull));
    // (3) uniforms with few significant bits (small (h >> 11), large exponents)
    xs[3] = (double)((h >> 11) >> (h & 63)) * 0x1p-53 + 0x1p-54;
    for (int c = 0; c < 4; ++c) {
      const double a = gmk::glibc_log_t(xs[c], tab), b = std::log(xs[c]);
      near1 += gmk::glibc_log_is_near1(xs[c]);
      if (gmk::glog_bits(a) != gmk::glog_bits(b)) {
        if (bad[c] < 3) fprintf(stderr, "class %d x=%a clone=%a libm=%a\n", c, xs[c], a, b);
        ++bad[c];
      }
    }
  }
  printf("%lld %lld %lld %lld %lld %lld\n", bad[0], bad[1], bad[2], bad[3], n, near1);
  return (bad[0] | bad[1] | bad[2] | bad[3]) ? 1 : 0;
}
