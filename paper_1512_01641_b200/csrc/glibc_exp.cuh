// glibc_exp.cuh -- bit-exact device restatement of the host's math.exp.
//
// The reference's logistic calls math.exp (classifier.py:145-147), i.e.
// glibc 2.39 libm `exp`, which dispatches (IFUNC) to __exp_fma on hosts
// with FMA+AVX2: sysdeps/ieee754/dbl-64/e_exp.c compiled with -mfma.
// glibc's exp is not correctly rounded (about 1 in 1200 results differs
// from the correctly rounded value), so CUDA's exp() cannot be used.
// This is the same algorithm -- 128-entry 2^(k/N) table, degree-5
// polynomial -- with every FMA placed exactly where GCC contracted the
// glibc source in the host binary (libm.so.6 .text at 0x79b60, read with
// objdump), and every other operation a separate IEEE op:
//
//   kd   = fma(x, InvLn2N, Shift);  ki = bits(kd);  kd -= Shift
//   r    = fma(kd, NegLn2loN, fma(kd, NegLn2hiN, x))
//   tmp  = fma(r2*r2, fma(r, C5, C4), fma(fma(r, C3, C2), r2, r + tail))
//   exp  = fma(scale, tmp, scale)
//
// plus the |x| in [512, 1024) special case (scale*tmp then + scale, no
// FMA there) and the tiny / huge / non-finite branches.  Compiles for the
// host too (std::fma), so CPU tests can check it against libm directly.
//
// Attribution: the algorithm, its constants and its operation order are
// those of the GNU C Library's exp (sysdeps/ieee754/dbl-64/e_exp.c,
// e_exp_data.c, math_config.h; Copyright (C) 2018-2024 Free Software
// Foundation, Inc., originally contributed by Szabolcs Nagy / Arm Ltd.),
// licensed under the GNU Lesser General Public License v2.1 or later.
// Reproducing that exact operation order is what makes the device result
// bit-identical to the reference's math.exp.
#pragma once

#include <stdint.h>
#include <string.h>
#include <math.h>

#if defined(__CUDACC__)
#define BIMINE_HD __host__ __device__ __forceinline__
#else
#define BIMINE_HD static inline
#endif

namespace bimine {

BIMINE_HD double u2d(uint64_t u) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double((long long)u);
#else
  double d;
  memcpy(&d, &u, 8);
  return d;
#endif
}

BIMINE_HD uint64_t d2u(double d) {
#if defined(__CUDA_ARCH__)
  return (uint64_t)__double_as_longlong(d);
#else
  uint64_t u;
  memcpy(&u, &d, 8);
  return u;
#endif
}

// Separately rounded IEEE operations (never contracted).
BIMINE_HD double fadd(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dadd_rn(a, b);
#else
  return a + b;
#endif
}
BIMINE_HD double fsub(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dsub_rn(a, b);
#else
  return a - b;
#endif
}
BIMINE_HD double fmul(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dmul_rn(a, b);
#else
  return a * b;
#endif
}
BIMINE_HD double fdiv(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __ddiv_rn(a, b);
#else
  return a / b;
#endif
}
BIMINE_HD double ffma(double a, double b, double c) {
#if defined(__CUDA_ARCH__)
  return __fma_rn(a, b, c);
#else
  return fma(a, b, c);
#endif
}

static const uint64_t kExpTable[256] = {
#include "exp_table.inc"
};

// exp_data scalars (glibc e_exp_data.c; identical to the values at
// libm.so.6 .rodata 0xb4980..0xb49b8 on the build image).
#define BIMINE_EXP_INVLN2N 0x1.71547652b82fep+7
#define BIMINE_EXP_SHIFT 0x1.8p52
#define BIMINE_EXP_NEGLN2HIN (-0x1.62e42fefa0000p-8)
#define BIMINE_EXP_NEGLN2LON (-0x1.cf79abc9e3b3ap-47)
#define BIMINE_EXP_C2 0x1.ffffffffffdbdp-2
#define BIMINE_EXP_C3 0x1.555555555543cp-3
#define BIMINE_EXP_C4 0x1.55555cf172b91p-5
#define BIMINE_EXP_C5 0x1.1111167a4d017p-7

// `tab` is the 256-entry table in any address space the caller prefers
// (shared memory inside the score kernel, global/constant elsewhere).
BIMINE_HD double glibc_exp(double x, const uint64_t *tab) {
  const uint64_t ix = d2u(x);
  uint32_t abstop = (uint32_t)(ix >> 52) & 0x7ffu;
  if (abstop - 0x3c9u > 0x3eu) {  // |x| < 2^-54 or |x| >= 512 or non-finite
    if ((int32_t)(abstop - 0x3c9u) < 0) return fadd(x, 1.0);  // tiny: 1 + x
    if (abstop > 0x408u) {                                    // |x| >= 1024
      if (ix == 0xfff0000000000000ull) return 0.0;
      if (abstop == 0x7ffu) return fadd(x, 1.0);  // +inf, nan
      return (ix >> 63) ? 0.0 : u2d(0x7ff0000000000000ull);
    }
    abstop = 0;  // 512 <= |x| < 1024: finish in the special case below
  }
  double kd = ffma(x, BIMINE_EXP_INVLN2N, BIMINE_EXP_SHIFT);
  const uint64_t ki = d2u(kd);
  kd = fsub(kd, BIMINE_EXP_SHIFT);
  double r = ffma(kd, BIMINE_EXP_NEGLN2HIN, x);
  r = ffma(kd, BIMINE_EXP_NEGLN2LON, r);
  const uint32_t idx = 2u * (uint32_t)(ki & 127u);
  const double tail = u2d(tab[idx]);
  uint64_t sbits = tab[idx + 1] + (ki << 45);
  const double p1 = ffma(r, BIMINE_EXP_C3, BIMINE_EXP_C2);
  const double rt = fadd(r, tail);
  const double r2 = fmul(r, r);
  const double p2 = ffma(r, BIMINE_EXP_C5, BIMINE_EXP_C4);
  const double q = ffma(p1, r2, rt);
  const double r4 = fmul(r2, r2);
  const double tmp = ffma(r4, p2, q);
  if (abstop != 0) {
    const double scale = u2d(sbits);
    return ffma(scale, tmp, scale);
  }
  // specialcase (e_exp.c): result would over/underflow the scale bits
  if ((ki & 0x80000000ull) == 0) {  // k > 0
    sbits -= 1009ull << 52;
    const double scale = u2d(sbits);
    return fmul(ffma(scale, tmp, scale), 0x1p1009);
  }
  sbits += 1022ull << 52;  // k < 0
  const double scale = u2d(sbits);
  const double st = fmul(tmp, scale);
  double y = fadd(scale, st);
  if (1.0 > y) {  // subnormal result: round once, then scale
    const double hi = fadd(y, 1.0);
    double lo = fadd(fsub(scale, y), st);
    double t = fadd(fadd(fsub(1.0, hi), y), lo);
    y = fsub(fadd(t, hi), 1.0);
    if (y == 0.0) y = 0.0;
  }
  return fmul(y, 0x1p-1022);
}

}  // namespace bimine
