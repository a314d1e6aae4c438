// Bit-exact restatement of the three glibc libm routines the reference's trace
// generator calls (workload.cpp:19-28, 58: std::log, std::cos, std::exp), as
// glibc 2.39 runs them on x86-64 hosts with FMA+AVX2: the IFUNC selects the
// FMA builds of sysdeps/ieee754/dbl-64 e_exp.c / e_log.c (ARM optimized
// routines) and s_sin.c (IBM Accurate Mathematical Library), so every a*b+c
// that GCC contracted in those builds is one fused multiply-add here and
// every other operation is one IEEE-rounded op — the operation sequence was
// read off the FMA entry points' disassembly (scripts/extract_libm_tables.py
// names them), not re-derived from the C sources.  Data words (polynomials,
// tables) come from that libm build via glibc_libm_tables.h.
//
// Used on the device by the trace generator (gen.cu); the same header
// compiles as plain C++ for the CPU test that compares it with the host libm
// (tests/test_libm.py).  Domain notes: exp and log are complete for finite
// inputs; cos covers |x| < 105414350 (the generator only passes 2*pi*[0,1)),
// beyond which glibc switches to __branred — not restated, returns NaN.
#pragma once
#include <cstdint>
#include <cstring>
#include <cmath>

#if defined(__CUDACC__)
#define SBS_LIBM_HD __device__ __forceinline__
#ifndef SBS_LIBM_TABLE
#define SBS_LIBM_TABLE __device__ const
#endif
#else
#define SBS_LIBM_HD static inline
#ifndef SBS_LIBM_TABLE
#define SBS_LIBM_TABLE static const
#endif
#endif

#include "glibc_libm_tables.h"

namespace sbs {
namespace glibc {

SBS_LIBM_HD double as_d(uint64_t u) {
#ifdef __CUDA_ARCH__
  return __longlong_as_double((long long)u);
#else
  double d;
  std::memcpy(&d, &u, 8);
  return d;
#endif
}
SBS_LIBM_HD uint64_t as_u(double d) {
#ifdef __CUDA_ARCH__
  return (uint64_t)__double_as_longlong(d);
#else
  uint64_t u;
  std::memcpy(&u, &d, 8);
  return u;
#endif
}
// one rounding each (host: build with -ffp-contract=off)
SBS_LIBM_HD double f_fma(double a, double b, double c) {
#ifdef __CUDA_ARCH__
  return __fma_rn(a, b, c);
#else
  return std::fma(a, b, c);
#endif
}
SBS_LIBM_HD double f_mul(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dmul_rn(a, b);
#else
  return a * b;
#endif
}
SBS_LIBM_HD double f_add(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dadd_rn(a, b);
#else
  return a + b;
#endif
}
SBS_LIBM_HD double f_sub(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dsub_rn(a, b);
#else
  return a - b;
#endif
}
SBS_LIBM_HD double f_abs(double a) { return as_d(as_u(a) & 0x7fffffffffffffffull); }
SBS_LIBM_HD double f_neg(double a) { return as_d(as_u(a) ^ 0x8000000000000000ull); }
#define SBS_D(name) as_d(name)

// ---------------------------------------------------------------- exp
// e_exp.c: exp(x) = 2^(k/128) * exp(r); specialcase() for |x| in [512, 1024).
SBS_LIBM_HD double exp_special(double tmp, uint64_t sbits, uint64_t ki) {
  if ((ki & 0x80000000ull) == 0) {  // k > 0: the exponent of scale might overflow
    sbits -= 1009ull << 52;
    const double scale = as_d(sbits);
    return f_mul(f_fma(scale, tmp, scale), SBS_D(EXP_2P1009));
  }
  // k < 0: the result may be subnormal; round once in the final multiply
  sbits += 1022ull << 52;
  const double scale = as_d(sbits);
  const double st = f_mul(scale, tmp);
  double y = f_add(scale, st);
  if (y < 1.0) {
    const double lo = f_add(f_sub(scale, y), st);
    const double hi = f_add(y, 1.0);
    double t = f_add(f_sub(1.0, hi), y);
    t = f_add(t, lo);
    t = f_add(t, hi);
    y = f_sub(t, 1.0);
    if (y == 0.0) y = 0.0;
  }
  return f_mul(y, SBS_D(EXP_2PM1022));
}

SBS_LIBM_HD double exp(double x) {
  const uint64_t ix = as_u(x);
  uint32_t abstop = (uint32_t)(ix >> 52) & 0x7ffu;
  if (abstop - 0x3c9u > 0x3eu) {
    if ((int32_t)(abstop - 0x3c9u) < 0) return f_add(x, 1.0);  // |x| < 2^-54
    if (abstop > 0x408u) {                                      // |x| >= 1024
      if (ix == 0xfff0000000000000ull) return 0.0;
      if (abstop == 0x7ffu) return f_add(x, 1.0);
      return (ix >> 63) ? 0.0 : as_d(0x7ff0000000000000ull);  // __math_uflow / oflow
    }
    abstop = 0;  // large |x|: specialcase below
  }
  double kd = f_fma(x, SBS_D(EXP_INVLN2N), SBS_D(EXP_SHIFT));
  const uint64_t ki = as_u(kd);
  kd = f_sub(kd, SBS_D(EXP_SHIFT));
  double r = f_fma(kd, SBS_D(EXP_NEGLN2HIN), x);
  r = f_fma(kd, SBS_D(EXP_NEGLN2LON), r);
  const uint32_t idx = 2u * (uint32_t)(ki & 127u);
  const uint64_t top = ki << 45;
  const double tail = as_d(EXP_TAB[idx]);
  const uint64_t sbits = EXP_TAB[idx + 1] + top;
  const double t1 = f_fma(SBS_D(EXP_C3), r, SBS_D(EXP_C2));
  const double tr = f_add(r, tail);
  const double r2 = f_mul(r, r);
  const double t2 = f_fma(r, SBS_D(EXP_C5), SBS_D(EXP_C4));
  const double p = f_fma(t1, r2, tr);
  const double r4 = f_mul(r2, r2);
  const double tmp = f_fma(r4, t2, p);
  if (abstop == 0) return exp_special(tmp, sbits, ki);
  const double scale = as_d(sbits);
  return f_fma(scale, tmp, scale);
}

// ---------------------------------------------------------------- log
// e_log.c: log(x) = log1p(z/c - 1) + log(c) + k ln2, with the |x - 1| < ~0.065
// inputs on a separate polynomial.
SBS_LIBM_HD double log(double x) {
  uint64_t ix = as_u(x);
  if (ix - 0x3fee000000000000ull < 0x3090000000000ull) {
    if (ix == 0x3ff0000000000000ull) return 0.0;
    const double r = f_sub(x, 1.0);
    double a1 = f_fma(r, SBS_D(LOG_B2), SBS_D(LOG_B1));
    double a2 = f_fma(r, SBS_D(LOG_B5), SBS_D(LOG_B4));
    const double r2 = f_mul(r, r);
    const double a3 = f_fma(r, SBS_D(LOG_B8), SBS_D(LOG_B7));
    a1 = f_fma(r2, SBS_D(LOG_B3), a1);
    a2 = f_fma(r2, SBS_D(LOG_B6), a2);
    const double r3 = f_mul(r, r2);
    double q = f_fma(r2, SBS_D(LOG_B9), a3);
    q = f_fma(r3, SBS_D(LOG_B10), q);
    q = f_fma(q, r3, a2);
    q = f_fma(q, r3, a1);
    const double c27 = SBS_D(LOG_2P27);
    const double t = f_fma(r, c27, r);           // r + r*2^27
    const double rhi = f_fma(f_neg(c27), r, t);  // ... - r*2^27
    const double rhi2 = f_mul(rhi, rhi);
    const double rlo = f_sub(r, rhi);
    const double b0 = SBS_D(LOG_B0);
    const double hi = f_fma(rhi2, b0, r);
    double lo = f_sub(r, hi);
    const double rr = f_add(r, rhi);
    lo = f_fma(rhi2, b0, lo);
    lo = f_fma(f_mul(b0, rlo), rr, lo);
    const double y = f_fma(q, r3, lo);
    return f_add(hi, y);
  }
  const uint32_t top = (uint32_t)(ix >> 48);
  if (top - 0x10u > 0x7fdfu) {
    if ((ix << 1) == 0) return as_d(0xfff0000000000000ull);  // log(+-0) = -inf
    if (ix == 0x7ff0000000000000ull) return x;                // log(inf)
    if ((top & 0x8000u) || ((~top & 0x7ff0u) == 0)) return as_d(0x7ff8000000000000ull);
    ix = as_u(f_mul(x, 4503599627370496.0));  // subnormal: x * 2^52
    ix -= 52ull << 52;
  }
  const uint64_t tmp = ix - 0x3fe6000000000000ull;
  const uint32_t i = (uint32_t)(tmp >> 45) & 127u;
  const int32_t k = (int32_t)((int64_t)tmp >> 52);
  const uint64_t iz = ix - (tmp & 0xfff0000000000000ull);
  const double invc = as_d(LOG_TAB[2 * i]);
  const double logc = as_d(LOG_TAB[2 * i + 1]);
  const double z = as_d(iz);
  const double kd = (double)k;
  const double w = f_fma(kd, SBS_D(LOG_LN2HI), logc);
  const double r = f_fma(z, invc, -1.0);
  const double a12 = f_fma(r, SBS_D(LOG_A2), SBS_D(LOG_A1));
  const double hi = f_add(r, w);
  const double r2 = f_mul(r, r);
  double lo = f_add(f_sub(w, hi), r);
  lo = f_fma(kd, SBS_D(LOG_LN2LO), lo);
  const double r3 = f_mul(r, r2);
  const double a34 = f_fma(r, SBS_D(LOG_A4), SBS_D(LOG_A3));
  lo = f_fma(r2, SBS_D(LOG_A0), lo);
  const double p = f_fma(a34, r2, a12);
  const double y = f_fma(r3, p, lo);
  return f_add(y, hi);
}

// ---------------------------------------------------------------- cos
// s_sin.c: table-driven sin/cos of x + dx around the nearest multiple of
// 1/128 (__sincostab), Taylor for small arguments, Cody-Waite reduction by
// pi/2 (reduce_sincos) below 105414350.
SBS_LIBM_HD double sc_do_cos(double x, double dx) {  // do_cos; dx already sign-adjusted
  const double big = SBS_D(SC_BIG);
  const double ax = f_abs(x);
  const double u = f_add(ax, big);
  double xr = f_sub(ax, f_sub(u, big));
  const int kk = (int)((uint32_t)as_u(u) << 2);
  xr = f_add(xr, dx);
  const double xx = f_mul(xr, xr);
  const double p = f_fma(xx, SBS_D(SC_SN5), SBS_D(SC_SN3));
  const double s = f_fma(f_mul(xr, xx), p, xr);
  double c = f_fma(xx, SBS_D(SC_CS6), SBS_D(SC_CS4));
  c = f_fma(xx, c, SBS_D(SC_CS2));
  c = f_mul(xx, c);
  const double sn = as_d(SINCOSTAB[kk]), ssn = as_d(SINCOSTAB[kk + 1]);
  const double cs = as_d(SINCOSTAB[kk + 2]), ccs = as_d(SINCOSTAB[kk + 3]);
  double cor = f_fma(f_neg(s), ssn, ccs);
  cor = f_fma(f_neg(c), cs, cor);
  cor = f_fma(f_neg(s), sn, cor);
  return f_add(cs, cor);
}

SBS_LIBM_HD double sc_taylor_sin(double a, double da) {  // TAYLOR_SIN
  const double xx = f_mul(a, a);
  double p = f_fma(xx, SBS_D(SC_S5), SBS_D(SC_S4));
  p = f_fma(xx, p, SBS_D(SC_S3));
  p = f_fma(xx, p, SBS_D(SC_S2));
  p = f_fma(xx, p, SBS_D(SC_S1));
  const double h = f_mul(da, SBS_D(SC_CS2));  // 0.5 * da
  const double q = f_fma(p, a, f_neg(h));
  const double t = f_fma(xx, q, da);
  return f_add(a, t);
}

SBS_LIBM_HD double sc_do_sin(double a, double da) {  // do_sin
  const double ax = f_abs(a);
  if (ax < SBS_D(SC_TAYLOR_LIM)) return sc_taylor_sin(a, da);
  const double dx = (a <= 0.0) ? f_neg(da) : da;
  const double big = SBS_D(SC_BIG);
  const double u = f_add(ax, big);
  const double xr = f_sub(ax, f_sub(u, big));
  const int kk = (int)((uint32_t)as_u(u) << 2);
  const double xx = f_mul(xr, xr);
  const double p = f_fma(xx, SBS_D(SC_SN5), SBS_D(SC_SN3));
  const double t = f_fma(f_mul(xr, xx), p, dx);
  double c = f_fma(xx, SBS_D(SC_CS6), SBS_D(SC_CS4));
  c = f_fma(xx, c, SBS_D(SC_CS2));
  const double s = f_add(xr, t);
  c = f_fma(xr, dx, f_mul(xx, c));
  const double sn = as_d(SINCOSTAB[kk]), ssn = as_d(SINCOSTAB[kk + 1]);
  const double cs = as_d(SINCOSTAB[kk + 2]), ccs = as_d(SINCOSTAB[kk + 3]);
  double cor = f_fma(s, ccs, ssn);
  cor = f_fma(f_neg(c), sn, cor);
  cor = f_fma(s, cs, cor);
  const double res = f_add(sn, cor);
  return as_d((as_u(res) & 0x7fffffffffffffffull) | (as_u(a) & 0x8000000000000000ull));
}

SBS_LIBM_HD double cos(double x) {
  const uint32_t k = (uint32_t)(as_u(x) >> 32) & 0x7fffffffu;
  if (k < 0x3e400000u) return 1.0;                 // |x| < 2^-27
  if (k < 0x3feb6000u) {                            // |x| < 0.855469
    const double dx = (x < 0.0) ? as_d(0x8000000000000000ull) : 0.0;
    return sc_do_cos(x, dx);
  }
  if (k < 0x400368fdu) {                            // |x| < 2.426265
    const double y = f_sub(SBS_D(SC_HP0), f_abs(x));
    const double a = f_add(y, SBS_D(SC_HP1));
    const double da = f_add(f_sub(y, a), SBS_D(SC_HP1));
    return sc_do_sin(a, da);
  }
  if (k < 0x419921fbu) {                            // |x| < 105414350: reduce_sincos
    const double t = f_fma(x, SBS_D(SC_HPINV), SBS_D(SC_TOINT));
    const double xn = f_sub(t, SBS_D(SC_TOINT));
    const int n = (int)(as_u(t) & 3u);
    const double nxn = f_neg(xn);
    double y = f_fma(nxn, SBS_D(SC_MP1), x);
    y = f_fma(nxn, SBS_D(SC_MP2), y);
    const double t2 = f_fma(nxn, SBS_D(SC_PP3), y);
    double db = f_fma(nxn, SBS_D(SC_PP3), f_sub(y, t2));
    const double b = f_fma(nxn, SBS_D(SC_PP4), t2);
    db = f_add(db, f_fma(nxn, SBS_D(SC_PP4), f_sub(t2, b)));
    double res;
    if ((n & 1) == 0) {                             // (n + 1) odd: do_cos
      res = sc_do_cos(b, (b < 0.0) ? f_neg(db) : db);
    } else {
      res = sc_do_sin(b, db);
    }
    return ((n + 1) & 2) ? f_neg(res) : res;
  }
  return as_d(0x7ff8000000000000ull);  // __branred range / inf / nan: not restated
}

#undef SBS_D
}  // namespace glibc
}  // namespace sbs
