/*
 * bimine_b200.h -- C ABI of the B200 (sm_100a) sentence-alignment hot path.
 *
 * This is the drop-in boundary for the reference package `bimine`
 * (arXiv 1512.01641 reimplementation, /root/reference/pkg).  The
 * reference has exactly one native FFI, the Cython module `_nwcore`
 * that `bimine.kernels` binds at import time (kernels.py:17-31):
 *
 *   nw_fill(double[:, ::1] dp, const double[:, ::1] sim,
 *           double mismatch, double bonus, double gap)            _nwcore.pyx:19-36
 *   nw_fill_wavefront(dp, sim, mismatch, bonus, gap, int workers)  _nwcore.pyx:45-70
 *
 * `bimine_nw_fill` / `bimine_nw_fill_wavefront` below replace those two
 * entry points one for one (host pointers, caller-initialised boundary,
 * interior written in place).  The remaining entry points move the rest
 * of the north-star path -- the Python loops of align.py:102-129
 * (build_score_matrix), align.py:132-163 (_traceback) and
 * align.py:323-332 (filter_by_threshold) -- behind the same boundary as
 * batched device calls, so the Python host only tokenises and packs.
 *
 * Conventions
 *  - every function returns 0 on success or a negative BIMINE_E* code;
 *    nothing throws across the ABI; bimine_last_error() returns a
 *    thread-local message for the last failure on the calling thread.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *    stream).  Calls are stream ordered; *_host calls synchronise the
 *    stream before returning.
 *  - "dev" pointers are CUDA device pointers, "host" pointers are plain
 *    host memory (pinned memory makes the copies asynchronous-fast).
 *  - all floating point is IEEE binary64, round-to-nearest, with no
 *    contraction, reproducing CPython float arithmetic bit for bit.
 */
#ifndef BIMINE_B200_H
#define BIMINE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BIMINE_OK 0
#define BIMINE_E_ARG (-1)      /* invalid argument (shape, NULL, range)            */
#define BIMINE_E_CUDA (-2)     /* CUDA runtime error                                */
#define BIMINE_E_LIMIT (-3)    /* input exceeds a documented kernel capacity        */
#define BIMINE_E_NOMEM (-4)    /* allocation failed                                 */

/* Model layout: the 21 doubles of SimilarityModel (classifier.py:115-124)
 * in this order: weights[6], bias, sigmoid_a, sigmoid_b,
 * feature_means[6], feature_scales[6]. */
#define BIMINE_MODEL_DOUBLES 21

/* Packed batch of document pairs.  Sentences are tokenised on the host
 * (text.py:97-104) into joint-vocabulary ids; every source and target
 * token string maps to one id space, so `t in target.token_set`
 * (classifier.py:78) and `token_set & token_set` (classifier.py:94) are
 * integer equality.  Per sentence the host supplies len(tokens),
 * len(set(tokens)) and len(text) (SentenceProfile, classifier.py:34-47). */
typedef struct bimine_batch {
  int64_t n_pairs;
  int64_t n_sentences;
  int64_t n_tokens;
  const int32_t *tokens;       /* [n_tokens] ids, sentences back to back; with
                                  token_bytes == 3: 3 * n_tokens bytes, each id
                                  little-endian in 24 bits (ids < 2^24)          */
  const int64_t *sent_tok_off; /* [n_sentences] first token of each sentence      */
  const int32_t *sent_len;     /* [n_sentences] token count (>= 1)                */
  const int32_t *sent_uniq;    /* [n_sentences] distinct token count              */
  const int32_t *sent_chars;   /* [n_sentences] code points of the raw sentence   */
  const int64_t *pair_src;     /* [n_pairs] index of the pair's first source sent */
  const int32_t *pair_n;       /* [n_pairs] source sentence count N (>= 1)        */
  const int64_t *pair_tgt;     /* [n_pairs] index of the first target sentence    */
  const int32_t *pair_m;       /* [n_pairs] target sentence count M (>= 1)        */
  const int64_t *pair_sim_off; /* [n_pairs] offset of the row-major N x M block   */
  int32_t token_bytes;         /* 4 (or 0): int32 ids; 3: packed 24-bit ids (the
                                  upload of bimine_mine_host shrinks by a quarter) */
  int32_t sent_bytes;          /* 4 (or 0): sent_len / sent_uniq / sent_chars are
                                  int32; 2: uint16 (every value < 65536).  The
                                  narrow form is accepted by bimine_mine_host
                                  only (its sentence upload halves); the other
                                  entry points refuse it with BIMINE_E_ARG      */
} bimine_batch;

/* Bilingual dictionary in CSR form over source ids (Lexicon,
 * lexicon.py:22-59).  Only entries with p > 0 are kept: the reference
 * reads them only through `p > best` with best >= 0 (classifier.py:78)
 * and `p > 0.0` (classifier.py:58). */
typedef struct bimine_dict_view {
  int64_t n_rows;          /* source ids >= n_rows have no translations */
  int64_t n_entries;
  const int64_t *row_ptr;  /* [n_rows + 1]                               */
  const int32_t *tgt;      /* [n_entries] target ids                     */
  const double *prob;      /* [n_entries] probabilities, all > 0         */
} bimine_dict_view;

/* One mined match, filter_by_threshold's (float(sim[i, j]), i, j)
 * (align.py:323-332). */
typedef struct bimine_match {
  double score;
  int32_t i;
  int32_t j;
} bimine_match;

/* Opaque device-resident dictionary (one per device). */
typedef struct bimine_dict bimine_dict;

const char *bimine_last_error(void);
const char *bimine_version(void);

/* ---- B1: reference FFI replacement (_nwcore.pyx:19-36, :45-70) -------
 * dp:  host, (n+1) x (m+1) row-major, row 0 and column 0 initialised by
 *      the caller (kernels.py:42-48); the interior is written in place.
 * sim: host, n x m row-major, the already reversed matrix
 *      (kernels.py:55,70; align.py:166-167).
 * Bit-identical to the reference fill.  `workers` is accepted for
 * signature compatibility; the anti-diagonal split is the GPU's. */
int bimine_nw_fill(double *dp, const double *sim, int64_t n, int64_t m,
                   double mismatch, double bonus, double gap, void *stream);
int bimine_nw_fill_wavefront(double *dp, const double *sim, int64_t n,
                             int64_t m, double mismatch, double bonus,
                             double gap, int workers, void *stream);

/* ---- dictionary -----------------------------------------------------
 * COO host arrays (src, tgt, prob) in lexicon iteration order.  Entries
 * with !(p > 0) are dropped; a repeated (src, tgt) keeps the last value
 * (read_lexicon, lexicon.py:177).  Builds a CSR on the host and uploads
 * it to the current device. */
int bimine_dict_create(const int32_t *src, const int32_t *tgt,
                       const double *prob, int64_t n_entries,
                       bimine_dict **out);
int bimine_dict_destroy(bimine_dict *dict);
int bimine_dict_view_get(const bimine_dict *dict, bimine_dict_view *view_dev);
int64_t bimine_dict_entries(const bimine_dict *dict);

/* ---- batch plan -------------------------------------------------------
 * Host-side summary of a packed batch (host pointers in batch_host): the
 * maxima that size the kernels and the work the per-pair score kernel
 * does not take in its one-CTA-per-pair launch:
 *   tiles     pairs with N > 64 or M > 64: (pair, i0, j0) per 64x64 tile
 *   long ids  pairs with a sentence of more than 255 tokens (tiled
 *             fallback kernel)
 *   large ids pairs with N > 64 or M > 64, ascending (their NW runs on
 *             the cluster kernel; every other pair's on one warp)
 * work_host (capacity work_cap int64) receives 3 * n_tiles tile triples,
 * then n_long pair ids, then n_large pair ids, then the large pairs' (N, M);
 * plan->work_len is the length needed
 * (BIMINE_E_ARG if work_cap is smaller).  The caller uploads
 * work_host[0 : work_len] and sets plan->work to the device copy. */
typedef struct bimine_plan {
  int32_t max_n, max_m;        /* over all pairs                          */
  int32_t max_uniq, max_len;   /* over all sentences                      */
  int64_t n_tiles;             /* 64x64 tiles of large pairs              */
  int64_t n_long;              /* pairs for the fallback kernel           */
  int32_t long_max_n, long_max_m;
  int64_t n_large;             /* pairs not in the one-CTA-per-pair launch */
  int64_t n_cells;             /* extent of sim: max pair_sim_off + N * M  */
  int64_t work_len;            /* 3 * n_tiles + n_long + 3 * n_large      */
  const int64_t *work;         /* device copy of work_host (set by caller)*/
  const int64_t *work_host;    /* optional: the host array itself (the NW
                                  launch then sizes the large pairs'
                                  scratch without a device round trip)    */
} bimine_plan;

int bimine_plan_batch(const bimine_batch *batch_host, int64_t *work_host,
                      int64_t work_cap, bimine_plan *plan);

/* ---- score matrix (align.py:102-129) -------------------------------
 * batch_dev: every pointer in the struct is a device pointer.
 * model: host array of BIMINE_MODEL_DOUBLES.
 * plan: from bimine_plan_batch, with large_ids uploaded.  BIMINE_E_LIMIT
 *   if a sentence has more than 4096 distinct or 16384 total tokens.
 * sim_dev: output, written once, row-major per pair at pair_sim_off. */
int bimine_score_batch(const bimine_dict *dict, const double *model,
                       const bimine_batch *batch_dev, const bimine_plan *plan,
                       double *sim_dev, void *stream);

/* ---- the mining step (score + NW + filter, one call) --------------------
 * build_score_matrix + nw_align + filter_by_threshold for every pair of a
 * device batch under one setting: sim_dev receives the score matrices
 * (written once); then one NW + traceback + filter launch for the pairs of
 * at most 64x64 sentences (a warp each) and, if the plan lists large
 * pairs, one cluster launch for those.  Outputs as in
 * bimine_nw_mine_batch with n_settings = 1 (out_off_dev: capacity
 * min(N, M) slots per pair; score_dev optional). */
int bimine_mine_batch(const bimine_dict *dict, const double *model,
                      const bimine_batch *batch_dev, const bimine_plan *plan,
                      double gap, double threshold, double mismatch, double bonus,
                      double *sim_dev, const int64_t *out_off_dev,
                      bimine_match *matches_dev, int32_t *counts_dev,
                      double *score_dev, void *stream);

/* ---- NW + traceback + threshold filter --------------------------------
 * Problem p = pair * n_settings + s aligns pair `pair` under setting s
 * (gap[s], threshold[s]); mismatch/bonus are shared (MiningConfig,
 * align.py:73-90).  Fill on the reversed matrix (align.py:170-181),
 * traceback with the diag > source-gap > target-gap tie order
 * (align.py:132-163), emit Match steps with sim >= threshold
 * (align.py:323-332).
 *   out_off_dev[p]   : slot offset of problem p in matches_dev (capacity
 *                      min(N, M) slots per problem)
 *   counts_dev[p]    : number of matches emitted for problem p
 *   score_dev[p]     : dp_rev[N, M] (Alignment.score), may be NULL
 * All arrays are device pointers; gap/threshold are device arrays of
 * n_settings doubles; max_n / max_m (host scalars) bound N and M and
 * size the per-warp direction storage. */
int bimine_nw_mine_batch(const double *sim_dev, const int64_t *pair_sim_off,
                         const int32_t *pair_n, const int32_t *pair_m,
                         int64_t n_pairs, int32_t max_n, int32_t max_m,
                         int32_t n_settings,
                         const double *gap_dev, const double *threshold_dev,
                         double mismatch, double bonus,
                         const int64_t *out_off_dev, bimine_match *matches_dev,
                         int32_t *counts_dev, double *score_dev, void *stream);

/* Full step lists for nw_align / nw_align_wavefront (Alignment.steps):
 * step codes 0 = Match, 1 = GapSource, 2 = GapTarget in forward order,
 * capacity N + M per pair at step_off_dev[p]; n_steps_dev[p] = count. */
int bimine_nw_steps_batch(const double *sim_dev, const int64_t *pair_sim_off,
                          const int32_t *pair_n, const int32_t *pair_m,
                          int64_t n_pairs, int32_t max_n, int32_t max_m,
                          const double *gap_dev,
                          double mismatch, double bonus,
                          const int64_t *step_off_dev, uint8_t *steps_dev,
                          int32_t *n_steps_dev, double *score_dev,
                          void *stream);

/* Order-preserving compaction of per-problem match slots:
 * match_base_dev[p] = exclusive prefix sum of counts; compact_dev
 * receives the matches of problem 0, 1, ... back to back;
 * total_dev[0] = sum of counts. */
int bimine_compact_matches(const bimine_match *matches_dev,
                           const int64_t *out_off_dev,
                           const int32_t *counts_dev, int64_t n_problems,
                           int64_t *match_base_dev, bimine_match *compact_dev,
                           int64_t *total_dev, void *stream);

/* ---- tuning agreement (tuning.py:60-82) --------------------------------
 * For every problem q = pair * n_settings + s of a bimine_nw_mine_batch
 * call: candidate = its match slots (out_off_dev[q], counts_dev[q]) read
 * as (i, j); reference = ref_ij_dev[2 * ref_off_dev[pair] ...] int32
 * (i, j) pairs, ref_len_dev[pair] of them.  matched_dev[q] = Match steps
 * joining equal pairs in the NW alignment of the two lists (match +1,
 * mismatch -1, gap 1).  The agreement percentage and the empty-list rules
 * are applied by the caller.  max_k / max_r bound the list lengths. */
int bimine_agreement_batch(const bimine_match *matches_dev,
                           const int64_t *out_off_dev, const int32_t *counts_dev,
                           int64_t n_pairs, int32_t n_settings,
                           const int32_t *ref_ij_dev, const int64_t *ref_off_dev,
                           const int32_t *ref_len_dev, int32_t max_k,
                           int32_t max_r, int32_t *matched_dev, void *stream);

/* ---- end to end from host buffers (the e2e call) ----------------------
 * batch_host: host pointers.  Copies the packed batch to the device,
 * scores, aligns under one setting, filters, compacts and copies back.
 *   counts_host[n_pairs]        matches per pair
 *   matches_host[capacity]      compacted matches in pair order
 *   capacity >= sum over pairs of min(N, M)
 *   sim_host (optional, may be NULL): the score matrices.
 * Host buffers are read while the call runs; pageable ones are staged
 * through page-locked memory by the library.  The scoring starts before
 * the call has validated the batch and overlaps the uploads (each score
 * CTA bounds-checks its pair and waits for its data); an invalid batch is
 * still reported with the usual error and no results.  sent_tok_off is
 * rebuilt on the device as the exclusive sum of sent_len; when the
 * caller's offsets differ from that packed layout they are uploaded and
 * the scores computed again.  Calls on one device run one at a time (other
 * threads' calls wait inside). */
int bimine_mine_host(const bimine_dict *dict, const double *model,
                     const bimine_batch *batch_host, double gap,
                     double threshold, double mismatch, double bonus,
                     int32_t *counts_host, bimine_match *matches_host,
                     int64_t capacity, int64_t *total_host, double *sim_host,
                     void *stream);

/* Host memcpy of `bytes` from src to dst over the library's copy threads
 * (BIMINE_STAGE_THREADS helpers + the caller) with streaming stores -- the
 * copy bimine_mine_host stages pageable inputs with; for a caller that
 * fills its own page-locked staging (the tuning sweep's re-uploads). */
int bimine_host_copy(void *dst, const void *src, int64_t bytes);

/* ---- host tokenizer and joint vocabulary (text.py:97-104) ---------------
 * A vocabulary maps token strings (UTF-8 bytes) to dense int32 ids; one
 * vocabulary holds the dictionary's strings and every sentence token, so
 * id equality is string equality.  bimine_tokenize_batch tokenises n
 * sentences (buf[off[k] : off[k+1]]) with the reference's rules and
 * appends their ids to tokens[] (capacity cap); per sentence it writes
 * len(tokens), len(set(tokens)) and len(text) in code points.  ASCII text
 * and text of code points below U+0180 (Latin-1, Latin Extended-A) are
 * tokenised exactly; any other sentence gets len_out = -1 and is left to
 * the caller (Unicode lower()/split()).  Large batches are split over
 * BIMINE_HOST_THREADS threads; ids are assigned in first-occurrence order
 * whatever the thread count. */
typedef struct bimine_vocab bimine_vocab;
int bimine_vocab_create(bimine_vocab **out);
int bimine_vocab_destroy(bimine_vocab *vocab);
int64_t bimine_vocab_size(const bimine_vocab *vocab);
int bimine_vocab_add_batch(bimine_vocab *vocab, const char *buf,
                           const int64_t *off, int64_t n, int32_t *ids_out);
int bimine_vocab_word(const bimine_vocab *vocab, int32_t id, const char **ptr,
                      int64_t *len);
int bimine_tokenize_batch(bimine_vocab *vocab, const char *buf,
                          const int64_t *off, int64_t n, int32_t *tokens,
                          int64_t cap, int64_t *n_tokens, int32_t *len_out,
                          int32_t *uniq_out, int32_t *chars_out);
/* The same with sentence k at ptrs[k] (lens[k] bytes) -- e.g. the caller's
 * own string storage, no concatenated copy (the Python package passes the
 * characters of compact ASCII str objects in place, csrc/pyhost.c);
 * len_prefix[k] = sum of lens[0:k] for k in 0..n (sizes the thread
 * ranges). */
int bimine_tokenize_ptrs(bimine_vocab *vocab, const char *const *ptrs,
                         const int64_t *lens, int64_t n,
                         const int64_t *len_prefix, int32_t *tokens,
                         int64_t cap, int64_t *n_tokens, int32_t *len_out,
                         int32_t *uniq_out, int32_t *chars_out);
/* Like bimine_score_batch, and also writes the six features of every cell
 * (extract_features / features_from_profiles, classifier.py:62-112) to
 * features_dev[6 * (pair_sim_off + i * M + j) + k], k = token ratio,
 * source coverage, target coverage, mean best probability, char ratio,
 * shared-token overlap.  Pairs whose sentences exceed 255 tokens
 * (plan->n_long > 0) are refused with BIMINE_E_LIMIT. */
int bimine_features_batch(const bimine_dict *dict, const double *model, const bimine_batch *batch,
                          const bimine_plan *plan, double *sim_dev, double *features_dev, void *stream);

/* ---- lexicon EM -----------------------------
 * Replaces the EM loop of build_lexicon (lexicon.py:60-120): `iterations`
 * rounds over device arrays, bit-identical to the reference's float64
 * sums (see csrc/lexicon_em.cuh).  Inputs, all device pointers:
 *   tgt_off[n_pairs + 1], tgt_tok[..]: target-side token ids per pair;
 *   row_ptr[n_src + 1], row_tgt[E]: the support of every source id (all
 *     co-occurring target ids, sorted per row);
 *   prob[E]: in/out, initially 1 / row length (lexicon.py:92-94);
 *   alive[E]: in/out, 1 initially; 0 once an entry left its row;
 *   occ_ptr[n_src + 1], occ_pair[..]: the pair of every occurrence of each
 *     source id, in corpus order (pairs with an empty side removed).
 * Returns BIMINE_E_ARG if a round looked up a target its row no longer
 * holds (the reference raises KeyError there). */
int bimine_lexicon_em(const int32_t *tgt_off, const int32_t *tgt_tok, int64_t n_pairs, int32_t n_src,
                      const int64_t *row_ptr, const int32_t *row_tgt, int64_t n_entries, double *prob,
                      uint8_t *alive, const int64_t *occ_ptr, const int32_t *occ_pair, int32_t iterations,
                      void *stream);

/* ---- test hook -------------------------------------------------------
 * Device evaluation of the score_from_margin logistic's exp
 * (classifier.py:145-147, glibc __exp_fma restated) over n host doubles;
 * used by the parity tests to pin the device exp against host math.exp. */
int bimine_exp_device(const double *x_host, double *y_host, int64_t n);

#ifdef __cplusplus
}
#endif
#endif /* BIMINE_B200_H */
