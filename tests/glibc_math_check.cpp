// Host check of paper_2605_06921_b200/csrc/glibc_math.cuh against this
// process's libm (log, sincos -- the calls the reference's Rng::normal
// makes, rng.hpp:49-62).  Built and run by tests/test_glibc_math.py:
//   glibc_math_check <random_pairs> <sweep_ulps>
// Prints "mismatches <k> evaluations <n>" and exits 1 on any mismatch.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>

#include "glibc_math.cuh"

extern "C" void sincos(double, double*, double*);

static uint64_t bits(double d) {
  uint64_t u;
  std::memcpy(&u, &d, 8);
  return u;
}
static double from_bits(uint64_t u) {
  double d;
  std::memcpy(&d, &u, 8);
  return d;
}

static long bad = 0, total = 0;

static void check_log(double x) {
  ++total;
  const double a = std::log(x), b = mqo_glibc::glibc_log(x);
  if (bits(a) != bits(b) && bad++ < 8) std::printf("log(%a): libm %a here %a\n", x, a, b);
}
static void check_sincos(double x) {
  double s1, c1, s2, c2;
  sincos(x, &s1, &c1);
  mqo_glibc::glibc_sincos(x, &s2, &c2);
  total += 2;
  if (bits(s1) != bits(s2) && bad++ < 8) std::printf("sin(%a): libm %a here %a\n", x, s1, s2);
  if (bits(c1) != bits(c2) && bad++ < 8) std::printf("cos(%a): libm %a here %a\n", x, c1, c2);
}

int main(int argc, char** argv) {
  const long pairs = argc > 1 ? std::atol(argv[1]) : 1000000;
  const long sweep = argc > 2 ? std::atol(argv[2]) : 20000;
  // 1. Box-Muller draws: u = (r >> 11) 2^-53, theta = 2 pi u2
  std::mt19937_64 g(20250801);
  for (long i = 0; i < pairs; ++i) {
    const double u1 = static_cast<double>(g() >> 11) * 0x1.0p-53;
    const double u2 = static_cast<double>(g() >> 11) * 0x1.0p-53;
    if (u1 > 0.0) check_log(u1);
    check_sincos(2.0 * 3.141592653589793 * u2);
  }
  // 2. consecutive doubles around every branch boundary of both routines
  const double edges[] = {
      // log: near-1 window [1 - 2^-4, 1 + 0x1.09p-4), table cells, u1 extremes
      1.0 - 0x1p-4, 1.0, 1.0 + 0x1.09p-4, 0x1.6p-1, 0.5, 0x1p-53, 0.25, 0.75,
      // sincos: 2^-27, 0.126, 0.855469, 2.426265, pi/2 multiples (reduction), 2 pi
      0x1p-27, 0.126, from_bits(0x3feb600000000000ull), from_bits(0x400368fd00000000ull),
      1.5707963267948966, 3.141592653589793, 4.71238898038469, 6.283185307179586,
      0.7853981633974483, 2.356194490192345, 3.9269908169872414, 5.497787143782138};
  for (double e : edges) {
    const uint64_t b0 = bits(e);
    for (long d = -sweep; d <= sweep; ++d) {
      const double x = from_bits(b0 + static_cast<uint64_t>(d));
      if (!(x > 0.0) || !std::isfinite(x)) continue;
      if (x < 1.0) check_log(x);
      if (x < 7.0) check_sincos(x);
    }
  }
  // 3. the u1 grid near 1 (1 - k 2^-53) and near 0 (k 2^-53)
  for (long k = 1; k <= sweep; ++k) {
    check_log(1.0 - static_cast<double>(k) * 0x1.0p-53);
    check_log(static_cast<double>(k) * 0x1.0p-53);
    check_sincos(2.0 * 3.141592653589793 * (static_cast<double>(k) * 0x1.0p-53));
    check_sincos(2.0 * 3.141592653589793 * (1.0 - static_cast<double>(k) * 0x1.0p-53));
  }
  std::printf("mismatches %ld evaluations %ld\n", bad, total);
  return bad ? 1 : 0;
}
