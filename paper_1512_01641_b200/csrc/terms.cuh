// terms.cuh -- the per-cell model arithmetic (classifier.py:62-148).
//
// Every feature is a ratio of small integers except mean_best_prob
// (a float sum over a count), and every margin term is
//   term_k(f) = (w_k * (f - mean_k)) / scale_k          (classifier.py:139)
// evaluated with separately rounded binary64 ops.  Terms of integer
// ratios are tabulated once per model on the device with exactly that op
// sequence (TermTables: bit-identical values, a load instead of ~25 FP64
// ops per term); the two float divisions that remain per cell use
// div_cr(), a correctly rounded a/b from the correctly rounded
// reciprocal y = RN(1/b): two Markstein correction steps
//   q1 = q0 + (a - b q0) y,  q2 = q1 + (a - b q1) y        (exact residuals by FMA)
// q1 is faithful, so q2 = RN(a/b) (Markstein's theorem); results near
// overflow/underflow take the IEEE division instead.
#pragma once

#include "common.cuh"

namespace bimine {

constexpr int kTermDim = 128;      // integer-ratio tables: numerator, denominator < 128
constexpr int kCharDim = 512;      // char-ratio table: Cs, Ct < 512
constexpr int kRecipDim = 4096;    // RN(1/c) for c < 4096

struct TermTables {
  const double *t0;   // [Ls][Lt]   term0(min(Ls/Lt, 4))
  const double *t1;   // [Ls][c]    term1(c/Ls)
  const double *t2;   // [Lt][c]    term2(c/Lt)
  const double *t5;   // [u][sh]    term5(sh/u)
  const double *t4;   // [Cs][Ct]   term4(min(Cs/Ct, 4))
  const double *rc;   // [c]        RN(1/c)
  const double *misc; // [0] term3(0.0), [1] RN(1/scale_3)
};

__device__ __forceinline__ double term(const Model &md, int k, double f) {
  return fdiv(fmul(md.w[k], fsub(f, md.mean[k])), md.scale[k]);
}

__device__ __forceinline__ double clip4(double r) { return (4.0 < r) ? 4.0 : r; }

__device__ __forceinline__ double div_cr(double a, double b, double y) {
  double q = fmul(a, y);
  double r = ffma(-q, b, a);
  q = ffma(r, y, q);
  r = ffma(-q, b, a);
  q = ffma(r, y, q);
  const double aq = fabs(q);
  if (!(aq <= 0x1p1000 && (aq >= 0x1p-960 || a == 0.0))) q = fdiv(a, b);
  return q;
}

__global__ void build_term_tables(const Model md, double *t0, double *t1, double *t2, double *t5, double *t4,
                                  double *rc, double *misc) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t D2 = (int64_t)kTermDim * kTermDim;
  if (tid < D2) {
    const int hi = (int)(tid / kTermDim), lo = (int)(tid % kTermDim);
    // hi = denominator-ish row, lo = column
    t0[tid] = (hi >= 1 && lo >= 1) ? term(md, 0, clip4(fdiv((double)hi, (double)lo))) : 0.0;
    t1[tid] = (hi >= 1 && lo <= hi) ? term(md, 1, fdiv((double)lo, (double)hi)) : 0.0;
    t2[tid] = (hi >= 1 && lo <= hi) ? term(md, 2, fdiv((double)lo, (double)hi)) : 0.0;
    t5[tid] = (hi >= 1 && lo <= hi) ? term(md, 5, fdiv((double)lo, (double)hi)) : 0.0;
  }
  const int64_t C2 = (int64_t)kCharDim * kCharDim;
  if (tid < C2) {
    const int cs = (int)(tid / kCharDim), ct = (int)(tid % kCharDim);
    t4[tid] = (cs >= 1 && ct >= 1) ? term(md, 4, clip4(fdiv((double)cs, (double)ct))) : 0.0;
  }
  if (tid < kRecipDim) rc[tid] = tid >= 1 ? fdiv(1.0, (double)tid) : 0.0;
  if (tid == 0) {
    misc[0] = term(md, 3, 0.0);
    misc[1] = fdiv(1.0, md.scale[3]);
  }
}

// One cell: features -> margin -> logistic, bit-identical to
// score_from_margin(margin(features_from_profiles(...))).
// rct = RN(1/Ct) (used only outside the char table).
// kInTables: the caller guarantees Ls, Lt, max(Us, Ut) < kTermDim and
// Cs, Ct < kCharDim (checked once per block), so every integer-ratio term
// is a table load
template <bool kInTables = false>
__device__ __forceinline__ double cell_score_t(const Model &md, const TermTables &T, int Ls, int Us, int Cs, int Lt,
                                               int Ut, int Ct, int cov, double sum, int covt, int sh,
                                               const uint64_t *tab) {
  const double t0 = (kInTables || (Ls < kTermDim && Lt < kTermDim)) ? T.t0[Ls * kTermDim + Lt]
                                                     : term(md, 0, clip4(fdiv((double)Ls, (double)Lt)));
  const double t1 = (kInTables || Ls < kTermDim) ? T.t1[Ls * kTermDim + cov]
                                                 : term(md, 1, fdiv((double)cov, (double)Ls));
  const double t2 = (kInTables || Lt < kTermDim) ? T.t2[Lt * kTermDim + covt]
                                                 : term(md, 2, fdiv((double)covt, (double)Lt));
  double t3;
  if (cov) {
    const double f3 = (kInTables || cov < kRecipDim) ? div_cr(sum, (double)cov, T.rc[cov]) : fdiv(sum, (double)cov);
    t3 = div_cr(fmul(md.w[3], fsub(f3, md.mean[3])), md.scale[3], T.misc[1]);
  } else {
    t3 = T.misc[0];
  }
  const double t4 = (kInTables || (Cs < kCharDim && Ct < kCharDim)) ? T.t4[Cs * kCharDim + Ct]
                                                     : term(md, 4, clip4(fdiv((double)Cs, (double)Ct)));
  const int u = Us > Ut ? Us : Ut;
  const double t5 = (kInTables || u < kTermDim) ? T.t5[u * kTermDim + sh]
                                                : term(md, 5, fdiv((double)sh, (double)u));
  double d = md.bias;
  d = fadd(d, t0);
  d = fadd(d, t1);
  d = fadd(d, t2);
  d = fadd(d, t3);
  d = fadd(d, t4);
  d = fadd(d, t5);
  const double z = fadd(fmul(md.a, d), md.b);
  // one exp and one division for both branches of score_from_margin:
  // z >= 0: exp(-z) / (1 + exp(-z)); z < 0: 1 / (1 + exp(z)); NaN takes
  // the z < 0 branch and its cut-off, as in Python
  const bool pos = z >= 0.0;
  double p;
  if (pos ? (z < 700.0) : (z > -700.0)) {
    const double e = glibc_exp(pos ? -z : z, tab);
    p = fdiv(pos ? e : 1.0, fadd(1.0, e));
  } else {
    p = pos ? 0.0 : 1.0;
  }
  if (0.0 > p) p = 0.0;
  if (1.0 < p) p = 1.0;
  return p;
}

}  // namespace bimine
