// lexicon_em.cuh -- EM estimation of the translation lexicon (SURVEY.md
// section 8 f4): build_lexicon, reference lexicon.py:60-120.
//
// One EM round, restated over integer ids:
//   for each sentence pair (in order), for each source occurrence s (in order):
//     denom = sum_j prob[s][t_j]            (sequential over target positions j)
//     if denom > 0: counts[s][t_j] += prob[s][t_j] / denom   for j in order
//   then per source word: total = Python's sum() (Neumaier-compensated in
//   CPython >= 3.12) of counts[s][.] in the order each target was first
//   counted this round (dict insertion order), and
//   prob[s][t] = counts[s][t] / total for every counted t (targets never
//   counted leave the row); rows never counted keep their probabilities.
//
// Every count of a source word s is written by the warp that owns s, which
// walks the occurrences of s in corpus order -- so each float64 sum is the
// reference's sequential sum.  Within one occurrence the target positions
// are spread over lanes; repeated targets are added in position order by
// the lowest lane of their group.  Rows are CSR over source ids with target
// ids sorted (binary search); `first` / `order` record the insertion order.
#pragma once

#include "common.cuh"

namespace bimine {

struct EmArgs {
  const int32_t *tgt_off;  // [pairs + 1] target tokens of pair p: tgt_tok[tgt_off[p] .. tgt_off[p+1])
  const int32_t *tgt_tok;
  int32_t n_src;           // source words
  const int64_t *row_ptr;  // [n_src + 1] entries of source word s
  const int32_t *row_tgt;  // [E] target id, sorted within a row
  double *prob;            // [E] in/out
  uint8_t *alive;          // [E] in/out: 0 once an entry left its row
  const int64_t *occ_ptr;  // [n_src + 1] occurrences of s, corpus order
  const int32_t *occ_pair; // [occurrences] sentence pair of each
  double *cnt;             // [E] scratch, zeroed per round
  int32_t *first;          // [E] scratch, -1 per round: rank of first count in its row
  int32_t *order;          // [E] scratch: row-local insertion order -> entry
  int32_t *status;         // [1] nonzero: a target without an entry (KeyError in the reference)
};

constexpr int kEmWarps = 8;

__device__ __forceinline__ int64_t em_find(const int32_t *__restrict__ tg, int64_t lo, int64_t hi, int32_t t) {
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    const int32_t v = __ldg(tg + mid);
    if (v < t) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(kEmWarps * 32) lexicon_em_round(const EmArgs A) {
  __shared__ double vbuf[kEmWarps][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  for (int s = blockIdx.x * kEmWarps + warp; s < A.n_src; s += gridDim.x * kEmWarps) {
    const int64_t r0 = A.row_ptr[s], r1 = A.row_ptr[s + 1];
    int32_t seen = 0;  // targets counted so far this round (warp-uniform)
    for (int64_t o = A.occ_ptr[s]; o < A.occ_ptr[s + 1]; ++o) {
      const int p = A.occ_pair[o];
      const int32_t tb = A.tgt_off[p], Lt = A.tgt_off[p + 1] - tb;
      // denom: sequential over the target positions
      double denom = 0.0;
      for (int c0 = 0; c0 < Lt; c0 += 32) {
        const int j = c0 + lane;
        double v = 0.0;
        if (j < Lt) {
          const int32_t t = __ldg(A.tgt_tok + tb + j);
          const int64_t r = em_find(A.row_tgt, r0, r1, t);
          if (r < r1 && __ldg(A.row_tgt + r) == t && A.alive[r]) v = A.prob[r];
          else atomicExch(A.status, 1);
        }
        vbuf[warp][lane] = v;
        __syncwarp();
        if (lane == 0) {
          const int n = min(32, Lt - c0);
          for (int k = 0; k < n; ++k) denom = fadd(denom, vbuf[warp][k]);
        }
        __syncwarp();
      }
      denom = __shfl_sync(kFull, denom, 0);
      if (!(denom > 0.0)) continue;  // reference: `if denom <= 0.0: continue`
      // counts, in position order
      for (int c0 = 0; c0 < Lt; c0 += 32) {
        const int j = c0 + lane;
        const bool act = j < Lt;
        int64_t r = -1;
        double x = 0.0;
        if (act) {
          const int32_t t = __ldg(A.tgt_tok + tb + j);
          r = em_find(A.row_tgt, r0, r1, t);
          x = fdiv(A.prob[r], denom);
        }
        const unsigned peers = __match_any_sync(kFull, act ? (long long)r : -1ll);
        const bool leader = act && (__ffs(peers) - 1) == lane;
        // first count of this target in this round: rank in insertion order
        const bool fresh = leader && A.first[r] < 0;
        const unsigned fb = __ballot_sync(kFull, fresh);
        if (fresh) {
          const int32_t rank = seen + __popc(fb & lt);
          A.first[r] = rank;
          A.order[r0 + rank] = (int32_t)(r - r0);
        }
        seen += __popc(fb);
        // the group's adds, in position order (usually a group of one)
        unsigned rest = peers;
        double acc = 0.0;
        if (leader) acc = A.cnt[r];
        while (rest) {
          const int k = __ffs(rest) - 1;
          rest &= rest - 1u;
          const double xk = __shfl_sync(peers, x, k);
          if (leader) acc = fadd(acc, xk);
        }
        if (leader) A.cnt[r] = acc;
        __syncwarp();
      }
    }
    // normalise: total = Python's sum() of the counts in insertion order --
    // CPython >= 3.12 sums floats with Neumaier's compensation
    // (bltinmodule.c): 0 + x0, compensated steps, + c when c is nonzero and
    // finite -- then counted targets get cnt / total
    if (seen > 0) {
      double total = 0.0;
      if (lane == 0) {
        double f = fadd(0.0, A.cnt[r0 + A.order[r0]]), c = 0.0;
        for (int32_t k = 1; k < seen; ++k) {
          const double x = A.cnt[r0 + A.order[r0 + k]];
          const double t = fadd(f, x);
          c = fadd(c, fabs(f) >= fabs(x) ? fadd(fsub(f, t), x) : fadd(fsub(x, t), f));
          f = t;
        }
        if (c != 0.0 && isfinite(c)) f = fadd(f, c);
        total = f;
      }
      total = __shfl_sync(kFull, total, 0);
      if (total > 0.0) {
        for (int64_t r = r0 + lane; r < r1; r += 32) {
          if (A.first[r] >= 0) {
            A.prob[r] = fdiv(A.cnt[r], total);
          } else {
            A.alive[r] = 0;  // not counted this round: the new row has no such target
            A.prob[r] = 0.0;
          }
        }
      }
    }
  }
}

}  // namespace bimine
