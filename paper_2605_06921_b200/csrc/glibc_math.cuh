// glibc_math.cuh -- bit-exact device replay of the host libm calls inside the
// reference's Box-Muller draw (Rng::normal, rng.hpp:49-62):
//
//     r = sqrt(-2 log u1);  theta = 2 pi u2;  spare = r sin(theta);  ... r cos(theta)
//
// The reference core is built with g++ -O3 (no -march), which fuses the
// sin/cos pair of one angle into a single sincos() call; on an x86-64 host
// with FMA + AVX2 the glibc 2.39 ifuncs resolve log -> __log_fma and
// sincos -> __sincos_fma (libm's own FMA build of sysdeps/ieee754/dbl-64
// e_log.c and s_sincos.c / s_sin.c).  CUDA's log/sincos differ from those in
// the last bit for a few percent of arguments, so the init noise would not
// match.  This header restates the two routines operation by operation --
// every add, multiply and fused multiply-add in the order and contraction
// the host binary executes them (read from its disassembly) -- so device
// and host produce identical bits.  IEEE-754 binary64 round-to-nearest
// add/sub/mul/fma are exactly specified, so the same operation sequence
// gives the same result on the GPU.
//
// Domains covered (all Box-Muller needs): glibc_log for positive normal x
// (u1 in [2^-53, 1)); glibc_sincos for |x| < 105414350 (theta in [0, 2 pi)).
// Outside them the functions return NaN rather than a wrong value.
//
// The data tables (__log_data, __sincostab) are generated from this image's
// libm.so.6 by scripts/gen_glibc_tables.py -> glibc_tables.inc.
// Validated against the host libm by tests/test_glibc_math.py (CPU, the
// functions compiled for the host) and tests/test_gpu_solver.py (device).
#pragma once
#include <cstdint>
#include <cstring>

#ifndef MQO_HD
#ifdef __CUDACC__
#define MQO_HD __host__ __device__ __forceinline__
#else
#define MQO_HD inline
#include <cmath>
#endif
#endif

namespace mqo_glibc {

#ifdef __CUDACC__
namespace dev {
#define MQO_GLIBC_TABLE __device__ static const
#include "glibc_tables.inc"
#undef MQO_GLIBC_TABLE
}  // namespace dev
#endif
namespace host {
#define MQO_GLIBC_TABLE static const
#include "glibc_tables.inc"
#undef MQO_GLIBC_TABLE
}  // namespace host

MQO_HD const uint64_t* log_const() {
#ifdef __CUDA_ARCH__
  return dev::kLogConst;
#else
  return host::kLogConst;
#endif
}
MQO_HD const uint64_t* log_tab() {
#ifdef __CUDA_ARCH__
  return dev::kLogTab;
#else
  return host::kLogTab;
#endif
}
MQO_HD const uint64_t* sincos_tab() {
#ifdef __CUDA_ARCH__
  return dev::kSinCosTab;
#else
  return host::kSinCosTab;
#endif
}

// exactly rounded primitives (no contraction possible across them)
MQO_HD double asd(uint64_t u) {
#ifdef __CUDA_ARCH__
  return __longlong_as_double(static_cast<long long>(u));
#else
  double d;
  std::memcpy(&d, &u, 8);
  return d;
#endif
}
MQO_HD uint64_t asu(double d) {
#ifdef __CUDA_ARCH__
  return static_cast<uint64_t>(__double_as_longlong(d));
#else
  uint64_t u;
  std::memcpy(&u, &d, 8);
  return u;
#endif
}
#ifdef __CUDA_ARCH__
MQO_HD double add(double a, double b) { return __dadd_rn(a, b); }
MQO_HD double sub(double a, double b) { return __dsub_rn(a, b); }
MQO_HD double mul(double a, double b) { return __dmul_rn(a, b); }
MQO_HD double fma(double a, double b, double c) { return __fma_rn(a, b, c); }
#else
// host build: compiled without -mfma / with -ffp-contract=off, so these stay
// separate roundings; std::fma is the correctly rounded fused operation
MQO_HD double add(double a, double b) { return a + b; }
MQO_HD double sub(double a, double b) { return a - b; }
MQO_HD double mul(double a, double b) { return a * b; }
MQO_HD double fma(double a, double b, double c) { return std::fma(a, b, c); }
#endif
MQO_HD double neg(double a) { return asd(asu(a) ^ 0x8000000000000000ull); }
MQO_HD double fabs_(double a) { return asd(asu(a) & 0x7fffffffffffffffull); }
MQO_HD double copysign_(double mag, double sgn) {
  return asd((asu(mag) & 0x7fffffffffffffffull) | (asu(sgn) & 0x8000000000000000ull));
}

// ------------------------------------------------------------------ log
// __log_fma (e_log.c, LOG_TABLE_BITS 7, the __FP_FAST_FMA branch).
MQO_HD double glibc_log(double x) {
  const uint64_t* C = log_const();
  const uint64_t ix = asu(x);
  if (ix - 0x3fee000000000000ull <= 0x308ffffffffffull) {  // x in [1 - 2^-4, 1 + 0x1.09p-4)
    if (ix == 0x3ff0000000000000ull) return 0.0;
    const double r = sub(x, 1.0);
    const double B0 = asd(C[7]);
    double p012 = fma(r, asd(C[9]), asd(C[8]));     // B1 + r B2
    double p345 = fma(r, asd(C[12]), asd(C[11]));   // B4 + r B5
    const double r2 = mul(r, r);
    const double p78 = fma(r, asd(C[15]), asd(C[14]));  // B7 + r B8
    p012 = fma(r2, asd(C[10]), p012);               // + r2 B3
    p345 = fma(r2, asd(C[13]), p345);               // + r2 B6
    const double r3 = mul(r, r2);
    double q = fma(r2, asd(C[16]), p78);            // + r2 B9
    q = fma(r3, asd(C[17]), q);                     // + r3 B10
    q = fma(q, r3, p345);
    q = fma(q, r3, p012);
    const double t = fma(r, 0x1p27, r);             // r + w, w = r 2^27
    const double rhi = fma(-0x1p27, r, t);          // (r + w) - w
    const double rhi2 = mul(rhi, rhi);
    const double rlo = sub(r, rhi);
    const double hi = fma(rhi2, B0, r);
    double lo = fma(rhi2, B0, sub(r, hi));
    const double s = add(r, rhi);
    lo = fma(mul(B0, rlo), s, lo);                  // lo += B0 rlo (rhi + r)
    const double y = fma(q, r3, lo);
    return add(hi, y);
  }
  const uint32_t top = static_cast<uint32_t>(ix >> 48);
  if (top - 0x0010u >= 0x7ff0u - 0x0010u) return asd(0x7ff8000000000000ull);  // not needed here
  const uint64_t tmp = ix - 0x3fe6000000000000ull;
  const int i = static_cast<int>((tmp >> 45) & 127);
  const int32_t k = static_cast<int32_t>(static_cast<int64_t>(tmp) >> 52);
  const uint64_t iz = ix - (tmp & 0xfff0000000000000ull);
  const uint64_t* T = log_tab();
  const double invc = asd(T[2 * i]), logc = asd(T[2 * i + 1]);
  const double z = asd(iz);
  const double kd = static_cast<double>(k);
  const double w = fma(kd, asd(C[0]), logc);        // k ln2hi + logc
  const double r = fma(z, invc, -1.0);
  const double p1 = fma(r, asd(C[4]), asd(C[3]));   // A1 + r A2
  const double hi = add(r, w);
  const double r2 = mul(r, r);
  double lo = add(sub(w, hi), r);
  lo = fma(kd, asd(C[1]), lo);                      // + k ln2lo
  const double r3 = mul(r, r2);
  const double p2 = fma(r, asd(C[6]), asd(C[5]));   // A3 + r A4
  lo = fma(r2, asd(C[2]), lo);                      // + r2 A0
  const double p = fma(p2, r2, p1);
  const double y = fma(r3, p, lo);
  return add(y, hi);
}

// --------------------------------------------------------------- sincos
// __sincos_fma (s_sincos.c with do_sin / do_cos / reduce_sincos of s_sin.c
// inlined).  Constants of s_sin.c / usncs.h:
constexpr double kSn3 = -0x1.5555555555515p-3, kSn5 = 0x1.11110e829872fp-7;
constexpr double kCs4 = -0x1.5555555555535p-5, kCs6 = 0x1.6c16bedd9e239p-10;
constexpr double kS1 = -0x1.5555555555555p-3, kS2 = 0x1.1111111110ecep-7;
constexpr double kS3 = -0x1.a01a019db08b8p-13, kS4 = 0x1.71de27b9a7ed9p-19;
constexpr double kS5 = -0x1.addffc2fcdf59p-26;
constexpr double kBig = 0x1.8p+45, kHp0 = 0x1.921fb54442d18p+0, kHp1 = 0x1.1a62633145c07p-54;
constexpr double kHpinv = 0x1.45f306dc9c883p-1, kToint = 0x1.8p+52;
constexpr double kMp1 = 0x1.921fb58000000p+0, kMp2 = -0x1.dde973c000000p-27;
constexpr double kPp3 = -0x1.cb3b398000000p-55, kPp4 = -0x1.d747f23e32ed7p-83;

struct SinCosRow {  // table row of |x| rounded to 1/128, and x - row
  double sn, ssn, cs, ccs, xr;
};
MQO_HD SinCosRow sincos_row(double ax) {
  const double u = add(ax, kBig);
  const int idx = static_cast<int>(static_cast<uint32_t>(asu(u)) << 2);
  const uint64_t* T = sincos_tab();
  return SinCosRow{asd(T[idx]), asd(T[idx + 1]), asd(T[idx + 2]), asd(T[idx + 3]),
                   sub(ax, sub(u, kBig))};
}
// TAYLOR_SIN(a*a, a, da): a + ((poly(xx) a - da/2) xx + da)
MQO_HD double taylor_sin(double a, double da) {
  const double xx = mul(a, a);
  double p = fma(xx, kS5, kS4);
  p = fma(xx, p, kS3);
  p = fma(xx, p, kS2);
  p = fma(xx, p, kS1);
  const double t1 = fma(p, a, neg(mul(da, 0.5)));
  return add(fma(xx, t1, da), a);
}
// do_sin body for |a| >= 0.126 on the row of |a| (dx already sign-adjusted)
MQO_HD double do_sin_row(const SinCosRow& w, double dx) {
  const double xr = w.xr;
  const double xx = mul(xr, xr);
  const double t = fma(mul(xx, xr), fma(xx, kSn5, kSn3), dx);
  const double s = add(t, xr);
  const double q = fma(fma(xx, kCs6, kCs4), xx, 0.5);
  const double c = fma(dx, xr, mul(xx, q));
  double cor = fma(s, w.ccs, w.ssn);
  cor = fma(neg(c), w.sn, cor);
  return add(fma(s, w.cs, cor), w.sn);
}
// do_cos body on the row of |a| with x = xr + dx
MQO_HD double do_cos_row(const SinCosRow& w, double dx) {
  const double xc = add(w.xr, dx);
  const double xx = mul(xc, xc);
  const double s = fma(mul(xc, xx), fma(xx, kSn5, kSn3), xc);
  const double c = mul(xx, fma(fma(xx, kCs6, kCs4), xx, 0.5));
  double cor = fma(neg(s), w.ssn, w.ccs);
  cor = fma(neg(c), w.cs, cor);
  cor = fma(neg(s), w.sn, cor);
  return add(w.cs, cor);
}

MQO_HD void glibc_sincos(double x, double* sinx, double* cosx) {
  const uint32_t k = static_cast<uint32_t>(asu(x) >> 32) & 0x7fffffffu;
  const double ax = fabs_(x);
  if (k <= 0x400368fcu) {
    if (k <= 0x3e3fffffu) {  // |x| < 2^-27
      *sinx = x;
      *cosx = 1.0;
      return;
    }
    if (k <= 0x3feb5fffu) {  // |x| < 0.855469: do_sin(x, 0), do_cos(x, 0)
      const SinCosRow w = sincos_row(ax);
      if (0.126 > ax) {
        const double xx = mul(x, x);
        double p = fma(xx, kS5, kS4);
        p = fma(xx, p, kS3);
        p = fma(xx, p, kS2);
        p = fma(xx, p, kS1);
        *sinx = add(x, fma(xx, fma(x, p, -0.0), 0.0));
      } else {
        const double dx = x > 0.0 ? 0.0 : -0.0;
        *sinx = copysign_(do_sin_row(w, dx), x);
      }
      *cosx = do_cos_row(w, x >= 0.0 ? 0.0 : -0.0);
      return;
    }
    // |x| < 2.426265: a + da = pi/2 - |x|; sin = copysign(do_cos(a, da), x),
    // cos = do_sin(a, da)
    const double y = sub(kHp0, ax);
    const double a = add(y, kHp1);
    const double da = add(sub(y, a), kHp1);
    const SinCosRow w = sincos_row(fabs_(a));
    *sinx = copysign_(do_cos_row(w, 0.0 > a ? neg(da) : da), x);
    if (0.126 > fabs_(a))
      *cosx = taylor_sin(a, da);
    else
      *cosx = copysign_(do_sin_row(w, a <= 0.0 ? neg(da) : da), a);
    return;
  }
  if (k > 0x419921fau) {  // needs __branred: outside the Box-Muller domain
    *sinx = *cosx = asd(0x7ff8000000000000ull);
    return;
  }
  // reduce_sincos: x = n pi/2 + (a + da)
  const double t = fma(x, kHpinv, kToint);
  const double xn = sub(t, kToint);
  const int n = static_cast<int>(asu(t) & 3);
  double y = fma(neg(xn), kMp1, x);
  y = fma(neg(xn), kMp2, y);
  const double t2 = fma(neg(xn), kPp3, y);
  const double db = fma(neg(xn), kPp3, sub(y, t2));
  double a = fma(neg(xn), kPp4, t2);
  double da = add(db, fma(neg(xn), kPp4, sub(t2, a)));
  if (n == 1 || n == 2) {
    a = neg(a);
    da = neg(da);
  }
  const SinCosRow w = sincos_row(fabs_(a));
  double s_val;
  if (0.126 > fabs_(a))
    s_val = taylor_sin(a, da);
  else
    s_val = copysign_(do_sin_row(w, 0.0 < a ? da : neg(da)), a);
  double c_val = do_cos_row(w, a < 0.0 ? neg(da) : da);
  if (n & 2) c_val = neg(c_val);
  if (n & 1) {
    *sinx = c_val;
    *cosx = s_val;
  } else {
    *sinx = s_val;
    *cosx = c_val;
  }
}

}  // namespace mqo_glibc
