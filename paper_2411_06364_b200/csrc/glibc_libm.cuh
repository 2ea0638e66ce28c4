// glibc_libm.cuh — glibc 2.39's exp and log, restated operation for operation
// so the device computes the same bits as the reference's std::exp / std::log.
//
// The reference's lognormal predictor is llround(true_rl * exp(N)) with N
// drawn by libstdc++'s polar method, which itself calls log (workload.hpp:
// 233-235, random.tcc:1811-1844). CUDA's exp/log are accurate but not
// glibc's: a 1-ulp difference next to a .5 boundary flips llround and
// changes the integer schedule. These ports follow the x86-64 FMA ifunc
// variants glibc selects on FMA+AVX2 hosts (__exp_fma / __log_fma: the ARM
// optimized-routines algorithms of sysdeps/ieee754/dbl-64/e_exp.c and
// e_log.c compiled with -mfma), including every place GCC contracted a
// multiply-add into an FMA — each fma() below is a vfmadd in that code, each
// separate * and + is a separate vmulsd / vaddsd. Tables: libm_tables.h
// (tools/gen_libm_tables.py). tests/test_libm_port.py checks both functions
// bit for bit against the host's libm over >1e8 inputs.
#pragma once
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "libm_tables.h"

#ifdef __CUDACC__
#define LMHD __host__ __device__ __forceinline__
#else
#define LMHD static inline
#endif

namespace econo_libm {

LMHD uint64_t as_u64(double x) {
#ifdef __CUDA_ARCH__
  return (uint64_t)__double_as_longlong(x);
#else
  uint64_t u;
  memcpy(&u, &x, 8);
  return u;
#endif
}
LMHD double as_f64(uint64_t u) {
#ifdef __CUDA_ARCH__
  return __longlong_as_double((long long)u);
#else
  double x;
  memcpy(&x, &u, 8);
  return x;
#endif
}
LMHD double dfma(double a, double b, double c) {
#ifdef __CUDA_ARCH__
  return __fma_rn(a, b, c);
#else
  return fma(a, b, c);
#endif
}
LMHD uint64_t exp_tab(int i) { return kExpTab[i]; }
LMHD double log_tab(int i) { return kLogTab[i]; }

// exp (e_exp.c): x = k ln2/N + r, exp(x) = 2^(k/N) * exp(r).
LMHD double exp(double x) {
  const uint64_t ix = as_u64(x);
  uint32_t abstop = (uint32_t)(ix >> 52) & 0x7ff;
  if (abstop - 0x3c9u > 0x3eu) {
    if ((int32_t)(abstop - 0x3c9u) < 0) return 1.0 + x;  // |x| < 2^-54
    if (abstop >= 0x409) {                                // |x| >= 1024 (or inf/nan)
      if (ix == 0xfff0000000000000ULL) return 0.0;        // -inf
      if (abstop == 0x7ff) return 1.0 + x;                // nan, +inf
      return (ix >> 63) ? 0x1p-767 * 0x1p-767 : 0x1p769 * 0x1p769;  // __math_uflow / __math_oflow
    }
    abstop = 0;  // large |x|: the scale may under/overflow, handled below
  }
  double kd = dfma(x, kExpInvLn2N, kExpShift);
  const uint64_t ki = as_u64(kd);
  kd = kd - kExpShift;
  double r = dfma(kd, kExpNegLn2hiN, x);
  r = dfma(kd, kExpNegLn2loN, r);
  const int idx = 2 * (int)(ki & 0x7f);
  const uint64_t top = ki << 45;
  const double p23 = dfma(r, kExpC3, kExpC2);
  const double tail_r = r + as_f64(exp_tab(idx));
  uint64_t sbits = exp_tab(idx + 1) + top;
  const double r2 = r * r;
  const double p45 = dfma(r, kExpC5, kExpC4);
  double tmp = dfma(p23, r2, tail_r);
  tmp = dfma(r2 * r2, p45, tmp);
  if (abstop == 0) {  // specialcase (e_exp.c)
    if ((ki & 0x80000000) == 0) {  // k > 0: the exponent of scale might have overflowed
      sbits -= 1009ULL << 52;
      const double scale = as_f64(sbits);
      return 0x1p1009 * dfma(scale, tmp, scale);
    }
    sbits += 1022ULL << 52;  // k < 0: keep the result's rounding exact in the subnormal range
    const double scale = as_f64(sbits);
    const double st = tmp * scale;
    double y = scale + st;
    if (y < 1.0) {
      const double hi = y + 1.0;
      double lo = (scale - y) + st;
      y = (((1.0 - hi) + y) + lo + hi) - 1.0;
      if (y == 0.0) y = 0.0;  // +0 (round-to-nearest)
    }
    return 0x1p-1022 * y;
  }
  const double scale = as_f64(sbits);
  return dfma(scale, tmp, scale);
}

// log (e_log.c): x = 2^k z, log(x) = k ln2 + log(c) + log1p(z/c - 1).
LMHD double log(double x) {
  uint64_t ix = as_u64(x);
  if (ix - 0x3fee000000000000ULL <= 0x308ffffffffffULL) {  // |x - 1| small: polynomial
    if (ix == 0x3ff0000000000000ULL) return 0.0;
    const double r = x - 1.0;
    double p1 = dfma(r, kLogB2, kLogB1);
    double p4 = dfma(r, kLogB5, kLogB4);
    const double r2 = r * r;
    double p7 = dfma(r, kLogB8, kLogB7);
    p1 = dfma(r2, kLogB3, p1);
    p4 = dfma(r2, kLogB6, p4);
    const double r3 = r * r2;
    double q = dfma(r2, kLogB9, p7);
    q = dfma(r3, kLogB10, q);
    q = dfma(q, r3, p4);
    q = dfma(q, r3, p1);
    const double t = dfma(r, 0x1p27, r);  // r + w, w = r * 2^27
    const double rhi = dfma(-0x1p27, r, t);  // vfnmadd: r + w - w
    const double rr = rhi * rhi;
    const double rlo = r - rhi;
    const double hi = dfma(rr, kLogB0, r);
    const double lo0 = dfma(rr, kLogB0, r - hi);
    const double lo = dfma(kLogB0 * rlo, r + rhi, lo0);
    return hi + dfma(q, r3, lo);
  }
  const uint32_t top = (uint32_t)(ix >> 48);
  if (top - 0x10u > 0x7fdfu) {
    if ((ix << 1) == 0) return -1.0 / 0.0;                  // log(+-0) = -inf
    if (ix == 0x7ff0000000000000ULL) return x;              // log(inf) = inf
    if ((top & 0x8000) || (top & 0x7ff0) == 0x7ff0) return (x - x) / (x - x);  // negative, nan
    ix = as_u64(x * 0x1p52) - (52ULL << 52);                // subnormal: normalize
  }
  const uint64_t tmp = ix - 0x3fe6000000000000ULL;
  const int i = (int)((tmp >> 45) & 0x7f);
  const int k = (int)((int64_t)tmp >> 52);
  const uint64_t iz = ix - (tmp & (0xfffULL << 52));
  const double invc = log_tab(2 * i), logc = log_tab(2 * i + 1);
  const double z = as_f64(iz);
  const double kd = (double)k;
  const double w = dfma(kd, kLogLn2hi, logc);
  const double r = dfma(z, invc, -1.0);
  const double a12 = dfma(r, kLogA2, kLogA1);
  const double hi = r + w;
  const double r2 = r * r;
  double lo = (w - hi) + r;
  lo = dfma(kd, kLogLn2lo, lo);
  const double rr2 = r * r2;
  const double a34 = dfma(r, kLogA4, kLogA3);
  lo = dfma(r2, kLogA0, lo);
  const double p = dfma(a34, r2, a12);
  return dfma(rr2, p, lo) + hi;
}

}  // namespace econo_libm
