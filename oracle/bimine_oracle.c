/*
 * bimine_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference `bimine` hot path
 * (/root/reference/pkg/src/bimine), used as the parity checker by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs.  The product path never links or calls it.
 *
 * Parity status: PINNED.  tests/test_oracle_golden.py checks this file
 * bit for bit against fixtures produced by running the reference itself
 * (tests/golden/make_golden.py imports /root/reference/pkg/src).
 *
 * Arithmetic: compiled with -O2 -ffp-contract=off and no -march, so
 * every + - * / is a separate IEEE binary64 operation exactly as CPython
 * evaluates the reference's float expressions; exp() is the host glibc
 * libm exp, i.e. the very function math.exp calls (classifier.py:145-147).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/bimine_b200.h"

#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------ */
/* classifier.py                                                       */
/* ------------------------------------------------------------------ */

static int cmp_i32(const void *a, const void *b) {
  int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
  return (x > y) - (x < y);
}

/* sorted unique copy; returns count */
static int32_t sorted_unique(const int32_t *ids, int32_t n, int32_t *out) {
  memcpy(out, ids, sizeof(int32_t) * (size_t)n);
  qsort(out, (size_t)n, sizeof(int32_t), cmp_i32);
  int32_t u = 0;
  for (int32_t k = 0; k < n; ++k)
    if (u == 0 || out[u - 1] != out[k]) out[u++] = out[k];
  return u;
}

static int contains(const int32_t *sorted, int32_t n, int32_t key) {
  int32_t lo = 0, hi = n;
  while (lo < hi) {
    int32_t mid = lo + (hi - lo) / 2;
    if (sorted[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  return lo < n && sorted[lo] == key;
}

/* _clip_ratio, classifier.py:50-51: min(numerator / denominator, 4.0);
 * Python min keeps the first argument unless the second is smaller. */
static double clip_ratio(int64_t num, int64_t den) {
  double r = (double)num / (double)den;
  return (4.0 < r) ? 4.0 : r;
}

typedef struct {
  const int32_t *tok; /* occurrence order */
  int32_t len;        /* len(tokens) */
  int32_t chars;      /* len(text)   */
  int32_t *set;       /* sorted unique ids */
  int32_t nset;       /* len(token_set) */
} profile_t;

/* reachable_targets, classifier.py:54-59 (sorted unique target ids). */
static int32_t reach_of(const bimine_dict_view *d, const profile_t *s,
                        int32_t **out) {
  int64_t cap = 0;
  for (int32_t k = 0; k < s->nset; ++k) {
    int32_t id = s->set[k];
    if (id >= 0 && id < d->n_rows) cap += d->row_ptr[id + 1] - d->row_ptr[id];
  }
  int32_t *buf = (int32_t *)malloc(sizeof(int32_t) * (size_t)(cap > 0 ? cap : 1));
  int32_t n = 0;
  for (int32_t k = 0; k < s->nset; ++k) {
    int32_t id = s->set[k];
    if (id < 0 || id >= d->n_rows) continue;
    for (int64_t e = d->row_ptr[id]; e < d->row_ptr[id + 1]; ++e)
      if (d->prob[e] > 0.0) buf[n++] = d->tgt[e];
  }
  int32_t *u = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  int32_t nu = sorted_unique(buf, n, u);
  free(buf);
  *out = u;
  return nu;
}

/* features_from_profiles, classifier.py:62-97. */
void oracle_features(const bimine_dict_view *d, const profile_t *src,
                     const profile_t *tgt, const int32_t *reach,
                     int32_t nreach, double f[6]) {
  double token_ratio = clip_ratio(src->len, tgt->len); /* :70 */
  double char_ratio = clip_ratio(src->chars, tgt->chars); /* :71 */

  int64_t covered = 0; /* :73-82, occurrence order, sequential sum */
  double best_prob_sum = 0.0;
  for (int32_t k = 0; k < src->len; ++k) {
    int32_t s = src->tok[k];
    double best = 0.0;
    if (s >= 0 && s < d->n_rows)
      for (int64_t e = d->row_ptr[s]; e < d->row_ptr[s + 1]; ++e) {
        double p = d->prob[e];
        if (contains(tgt->set, tgt->nset, d->tgt[e]) && p > best) best = p;
      }
    if (best > 0.0) {
      covered += 1;
      best_prob_sum += best;
    }
  }
  double source_coverage = (double)covered / (double)src->len; /* :83 */
  double mean_best_prob =
      covered ? best_prob_sum / (double)covered : 0.0; /* :84 */

  int64_t covered_target = 0; /* :88-92 */
  for (int32_t k = 0; k < tgt->len; ++k)
    if (contains(reach, nreach, tgt->tok[k])) covered_target += 1;
  double target_coverage = (double)covered_target / (double)tgt->len;

  int64_t shared = 0; /* :94-95, |set & set| / max(|set|, |set|) */
  for (int32_t a = 0, b = 0; a < src->nset && b < tgt->nset;) {
    if (src->set[a] == tgt->set[b]) { ++shared; ++a; ++b; }
    else if (src->set[a] < tgt->set[b]) ++a;
    else ++b;
  }
  int64_t den = src->nset > tgt->nset ? src->nset : tgt->nset;
  double overlap = (double)shared / (double)den;

  f[0] = token_ratio;
  f[1] = source_coverage;
  f[2] = target_coverage;
  f[3] = mean_best_prob;
  f[4] = char_ratio;
  f[5] = overlap;
}

/* SimilarityModel.margin, classifier.py:135-140 */
double oracle_margin(const double *model, const double *f) {
  const double *w = model, *mean = model + 9, *scale = model + 15;
  double d = model[6];
  for (int k = 0; k < 6; ++k) d += w[k] * (f[k] - mean[k]) / scale[k];
  return d;
}

/* SimilarityModel.score_from_margin, classifier.py:142-148 */
double oracle_score_from_margin(const double *model, double margin) {
  double z = model[7] * margin + model[8];
  double p;
  if (z >= 0) p = (z < 700) ? exp(-z) / (1.0 + exp(-z)) : 0.0;
  else p = (z > -700) ? 1.0 / (1.0 + exp(z)) : 1.0;
  double lo = (0.0 > p) ? 0.0 : p; /* max(p, 0.0) */
  return (1.0 < lo) ? 1.0 : lo;    /* min(., 1.0) */
}

void oracle_exp_array(const double *x, double *y, int64_t n) {
  for (int64_t k = 0; k < n; ++k) y[k] = exp(x[k]);
}

static void make_profile(const bimine_batch *b, int64_t sent, profile_t *p) {
  p->tok = b->tokens + b->sent_tok_off[sent];
  p->len = b->sent_len[sent];
  p->chars = b->sent_chars[sent];
  p->set = (int32_t *)malloc(sizeof(int32_t) * (size_t)(p->len > 0 ? p->len : 1));
  p->nset = sorted_unique(p->tok, p->len, p->set);
}

/* build_score_matrix, align.py:102-129, for pair `pair` of the batch.
 * out: row-major N x M. */
void oracle_score_pair(const bimine_dict_view *d, const double *model,
                       const bimine_batch *b, int64_t pair, double *out) {
  int32_t n = b->pair_n[pair], m = b->pair_m[pair];
  profile_t *tp = (profile_t *)malloc(sizeof(profile_t) * (size_t)m);
  for (int32_t j = 0; j < m; ++j) make_profile(b, b->pair_tgt[pair] + j, &tp[j]);
  for (int32_t i = 0; i < n; ++i) {
    profile_t sp;
    make_profile(b, b->pair_src[pair] + i, &sp);
    int32_t *reach;
    int32_t nreach = reach_of(d, &sp, &reach); /* hoisted per row, :125 */
    for (int32_t j = 0; j < m; ++j) {
      double f[6];
      oracle_features(d, &sp, &tp[j], reach, nreach, f);
      out[(int64_t)i * m + j] =
          oracle_score_from_margin(model, oracle_margin(model, f));
    }
    free(reach);
    free(sp.set);
  }
  for (int32_t j = 0; j < m; ++j) free(tp[j].set);
  free(tp);
}

/* ------------------------------------------------------------------ */
/* kernels.py / _nwcore.pyx / align.py                                 */
/* ------------------------------------------------------------------ */

/* kernels._init_table, kernels.py:42-48 */
void oracle_init_table(double *dp, int64_t n, int64_t m, double gap) {
  double ng = -gap;
  for (int64_t b = 0; b <= m; ++b) dp[b] = ng * (double)b;
  for (int64_t a = 1; a <= n; ++a) dp[a * (m + 1)] = ng * (double)a;
}

/* _nwcore.nw_fill, _nwcore.pyx:19-36 (row-major; the wavefront variant
 * :45-70 evaluates the identical per-cell expression). */
void oracle_nw_fill(double *dp, const double *sim, int64_t n, int64_t m,
                    double mismatch, double bonus, double gap) {
  int64_t w = m + 1;
  for (int64_t i = 1; i <= n; ++i)
    for (int64_t j = 1; j <= m; ++j) {
      double c = mismatch + sim[(i - 1) * m + (j - 1)] * (bonus - mismatch);
      double best = dp[(i - 1) * w + (j - 1)] + c;
      double cand = dp[(i - 1) * w + j] - gap;
      if (cand > best) best = cand;
      cand = dp[i * w + (j - 1)] - gap;
      if (cand > best) best = cand;
      dp[i * w + j] = best;
    }
}

/* _traceback, align.py:132-163.  steps: codes 0 Match / 1 GapSource /
 * 2 GapTarget; si/sj: the step's (i, j) (j = -1 / i = -1 when unused).
 * Returns the step count. */
int64_t oracle_traceback(const double *dp_rev, const double *sim, int64_t n,
                         int64_t m, double mismatch, double bonus, double gap,
                         uint8_t *steps, int32_t *si, int32_t *sj) {
  int64_t w = m + 1, k = 0, i = 0, j = 0;
  while (i < n && j < m) {
    double value = dp_rev[(n - i) * w + (m - j)];
    double c = mismatch + sim[i * m + j] * (bonus - mismatch);
    if (value == c + dp_rev[(n - i - 1) * w + (m - j - 1)]) {
      steps[k] = 0; si[k] = (int32_t)i; sj[k] = (int32_t)j; ++k; ++i; ++j;
    } else if (value == dp_rev[(n - i - 1) * w + (m - j)] - gap) {
      steps[k] = 1; si[k] = (int32_t)i; sj[k] = -1; ++k; ++i;
    } else {
      steps[k] = 2; si[k] = -1; sj[k] = (int32_t)j; ++k; ++j;
    }
  }
  while (i < n) { steps[k] = 1; si[k] = (int32_t)i; sj[k] = -1; ++k; ++i; }
  while (j < m) { steps[k] = 2; si[k] = -1; sj[k] = (int32_t)j; ++k; ++j; }
  return k;
}

/* nw_align, align.py:170-181: validate (caller), reverse, fill,
 * traceback.  Returns the step count; *score = dp_rev[-1, -1]. */
int64_t oracle_nw_align(const double *sim, int64_t n, int64_t m,
                        double mismatch, double bonus, double gap,
                        uint8_t *steps, int32_t *si, int32_t *sj,
                        double *score) {
  double *rev = (double *)malloc(sizeof(double) * (size_t)(n * m));
  for (int64_t a = 0; a < n; ++a)
    for (int64_t b = 0; b < m; ++b)
      rev[a * m + b] = sim[(n - 1 - a) * m + (m - 1 - b)]; /* :166-167 */
  double *dp = (double *)malloc(sizeof(double) * (size_t)((n + 1) * (m + 1)));
  oracle_init_table(dp, n, m, gap);
  oracle_nw_fill(dp, rev, n, m, mismatch, bonus, gap);
  int64_t k = oracle_traceback(dp, sim, n, m, mismatch, bonus, gap, steps, si, sj);
  *score = dp[(n + 1) * (m + 1) - 1];
  free(dp);
  free(rev);
  return k;
}

/* align_pair_indices for one pair of a packed batch (align.py:347-358):
 * build_score_matrix -> nw_align -> filter_by_threshold (:323-332).
 * out: capacity min(N, M).  Returns the match count. */
int64_t oracle_mine_pair(const bimine_dict_view *d, const double *model,
                         const bimine_batch *b, int64_t pair, double gap,
                         double threshold, double mismatch, double bonus,
                         bimine_match *out, double *sim_out) {
  int64_t n = b->pair_n[pair], m = b->pair_m[pair];
  double *sim = sim_out ? sim_out : (double *)malloc(sizeof(double) * (size_t)(n * m));
  oracle_score_pair(d, model, b, pair, sim);
  uint8_t *steps = (uint8_t *)malloc((size_t)(n + m));
  int32_t *si = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n + m));
  int32_t *sj = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n + m));
  double score;
  int64_t k = oracle_nw_align(sim, n, m, mismatch, bonus, gap, steps, si, sj, &score);
  int64_t c = 0;
  for (int64_t s = 0; s < k; ++s)
    if (steps[s] == 0) {
      double v = sim[(int64_t)si[s] * m + sj[s]];
      if (v >= threshold) {
        out[c].score = v; out[c].i = si[s]; out[c].j = sj[s]; ++c;
      }
    }
  free(steps); free(si); free(sj);
  if (!sim_out) free(sim);
  return c;
}

/* mine_corpus over a packed batch (align.py:402-448) with `threads`
 * OpenMP threads over pairs; per-pair results land in slot regions
 * out_off[p] (capacity min(N, M)), counts[p] = matches of pair p. */
void oracle_mine_batch(const bimine_dict_view *d, const double *model,
                       const bimine_batch *b, double gap, double threshold,
                       double mismatch, double bonus, const int64_t *out_off,
                       bimine_match *out, int32_t *counts, int threads) {
#ifdef _OPENMP
  if (threads < 1) threads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 4) num_threads(threads)
#endif
  for (int64_t p = 0; p < b->n_pairs; ++p)
    counts[p] = (int32_t)oracle_mine_pair(d, model, b, p, gap, threshold,
                                          mismatch, bonus, out + out_off[p], NULL);
  (void)threads;
}

/* score matrices only, OpenMP over pairs */
void oracle_score_batch(const bimine_dict_view *d, const double *model,
                        const bimine_batch *b, double *sim, int threads) {
#ifdef _OPENMP
  if (threads < 1) threads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 4) num_threads(threads)
#endif
  for (int64_t p = 0; p < b->n_pairs; ++p)
    oracle_score_pair(d, model, b, p, sim + b->pair_sim_off[p]);
  (void)threads;
}

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
