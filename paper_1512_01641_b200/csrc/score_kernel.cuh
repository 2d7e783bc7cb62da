// score_kernel.cuh -- the sentence-pair score matrix (build_score_matrix,
// align.py:102-129) as one sm_100a kernel.
//
// One CTA (8 warps) owns a tile of <= 64 source x <= 64 target sentences
// of one document pair (grid = pairs x ceil(N/64) x ceil(M/64)).  The
// target side of the tile is processed in chunks that fit the shared
// memory hash (<= cap_u distinct tokens, <= cap_t occurrences):
//
//  A  hash every target token of the chunk into a shared-memory open
//     addressing table -> dense id d; colmask[d] = 64-bit set of chunk
//     sentences containing d; per occurrence its d and a "first
//     occurrence in its sentence" bit (len(token_set) semantics).
//  B  for every source occurrence: srccol[d] |= bit(i) if the source
//     token itself is a chunk token (shared tokens, classifier.py:94);
//     for every dictionary translation t of it (p > 0): reachcol[d(t)]
//     |= bit(i) (reachable_targets, classifier.py:54-59).
//  C  warp per target sentence j, lanes over i: covered_target(i, j) =
//     sum over j's occurrences of bit i of reachcol (classifier.py:88-92)
//     and shared(i, j) = sum over j's first occurrences of bit i of
//     srccol (classifier.py:94).
//  D  warp per source sentence i, lanes over j: stream i's occurrences
//     in order, 32 at a time; each lane resolves one occurrence's
//     dictionary row against the chunk (candidates with their colmask),
//     then every lane walks the 32 records in order and, where its
//     target sentence holds a translation, takes the max probability and
//     adds it to the running sum -- the exact sequential sum of
//     classifier.py:75-82.  Finally the six features, the standardised
//     margin (classifier.py:135-140) and the logistic with glibc's exp
//     (classifier.py:142-148) in separately rounded binary64, and one
//     coalesced 8-byte store per cell.
#pragma once

#include "common.cuh"

namespace bimine {

constexpr int kScoreTile = 64;
constexpr int kScoreWarps = 8;
constexpr int kScoreThreads = kScoreWarps * 32;
constexpr int kCandInline = 4;
constexpr int kCntStride = 65;  // padded [i][j] count matrix (conflict free)

struct ScoreArgs {
  BatchDev b;
  DictDev d;
  Model md;
  double *sim;
  const int64_t *pair_ids;  // pairs of this launch (blockIdx.x indexes it); null = identity
  int cap_u;       // distinct target tokens per chunk
  int cap_t;       // target occurrences per chunk
  int hash_bits;   // log2(hash slots) = log2(2 * cap_u)
  int *status;     // BIMINE_E_LIMIT is written here if a sentence exceeds the caps
};

struct ScoreSmem {
  uint64_t *exp_tab;   // [256]
  uint64_t *colmask;   // [cap_u]
  uint64_t *reachcol;  // [cap_u]
  uint64_t *srccol;    // [cap_u]
  uint64_t *rec_any;   // [warps][32]
  uint64_t *rec_m;     // [warps][32][kCandInline]
  double *rec_p;       // [warps][32][kCandInline]
  int64_t *src_off;    // [64]
  int64_t *tgt_off;    // [64]
  uint32_t *cnt;       // [64][kCntStride]  covt | shared << 16
  uint32_t *first;     // [cap_t / 32]
  int32_t *keys;       // [2 cap_u]
  int32_t *src_len, *src_uniq, *src_chars;  // [64]
  int32_t *tgt_len, *tgt_uniq, *tgt_chars;  // [64]
  int32_t *tgt_occ0;   // [65]
  int32_t *rec_s;      // [warps][32]
  int32_t *misc;       // [4]: unique count, chunk end
  int16_t *dense;      // [2 cap_u]
  int16_t *occ_d;      // [cap_t]
  uint8_t *rec_nc;     // [warps][32]
};

__host__ __device__ inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Carves the dynamic shared memory; with base == nullptr returns the size.
__host__ __device__ inline size_t score_smem_layout(unsigned char *base, int cap_u, int cap_t, ScoreSmem *s) {
  size_t o = 0;
  auto take = [&](size_t bytes, size_t al) -> unsigned char * {
    o = align_up(o, al);
    unsigned char *p = base ? base + o : nullptr;
    o += bytes;
    return p;
  };
  ScoreSmem t;
  t.exp_tab = (uint64_t *)take(256 * 8, 16);
  t.colmask = (uint64_t *)take((size_t)cap_u * 8, 16);
  t.reachcol = (uint64_t *)take((size_t)cap_u * 8, 16);
  t.srccol = (uint64_t *)take((size_t)cap_u * 8, 16);
  t.rec_any = (uint64_t *)take(kScoreWarps * 32 * 8, 16);
  t.rec_m = (uint64_t *)take(kScoreWarps * 32 * kCandInline * 8, 16);
  t.rec_p = (double *)take(kScoreWarps * 32 * kCandInline * 8, 16);
  t.src_off = (int64_t *)take(64 * 8, 16);
  t.tgt_off = (int64_t *)take(64 * 8, 16);
  t.cnt = (uint32_t *)take(64 * kCntStride * 4, 16);
  t.first = (uint32_t *)take((size_t)(cap_t / 32 + 1) * 4, 16);
  t.keys = (int32_t *)take((size_t)cap_u * 2 * 4, 16);
  t.src_len = (int32_t *)take(64 * 4, 4);
  t.src_uniq = (int32_t *)take(64 * 4, 4);
  t.src_chars = (int32_t *)take(64 * 4, 4);
  t.tgt_len = (int32_t *)take(64 * 4, 4);
  t.tgt_uniq = (int32_t *)take(64 * 4, 4);
  t.tgt_chars = (int32_t *)take(64 * 4, 4);
  t.tgt_occ0 = (int32_t *)take(65 * 4, 4);
  t.rec_s = (int32_t *)take(kScoreWarps * 32 * 4, 4);
  t.misc = (int32_t *)take(4 * 4, 4);
  t.dense = (int16_t *)take((size_t)cap_u * 2 * 2, 4);
  t.occ_d = (int16_t *)take((size_t)cap_t * 2, 4);
  t.rec_nc = (uint8_t *)take(kScoreWarps * 32, 4);
  if (s) *s = t;
  return align_up(o, 16);
}

__device__ __forceinline__ int hash_find(const int32_t *keys, const int16_t *dense, int bits, int32_t key) {
  const uint32_t mask = (1u << bits) - 1u;
  uint32_t slot = hash_slot(key, 32 - bits);
  while (true) {
    const int32_t k = keys[slot];
    if (k == key) return dense[slot];
    if (k == -1) return -1;
    slot = (slot + 1u) & mask;
  }
}

__device__ __forceinline__ void hash_insert(int32_t *keys, int bits, int32_t key) {
  const uint32_t mask = (1u << bits) - 1u;
  uint32_t slot = hash_slot(key, 32 - bits);
  while (true) {
    const int32_t prev = atomicCAS(&keys[slot], -1, key);
    if (prev == -1 || prev == key) return;
    slot = (slot + 1u) & mask;
  }
}

// classifier.py:50-51, 62-97, 135-148 for one cell; every operation a
// separately rounded binary64 op in the reference's evaluation order.
__device__ __forceinline__ double cell_score(const Model &md, int Ls, int Us, int Cs, int Lt, int Ut, int Ct,
                                             int covered, double sum, int covt, int shared, const uint64_t *tab) {
  double f[6];
  f[0] = fdiv((double)Ls, (double)Lt);
  if (4.0 < f[0]) f[0] = 4.0;
  f[1] = fdiv((double)covered, (double)Ls);
  f[2] = fdiv((double)covt, (double)Lt);
  f[3] = covered ? fdiv(sum, (double)covered) : 0.0;
  f[4] = fdiv((double)Cs, (double)Ct);
  if (4.0 < f[4]) f[4] = 4.0;
  f[5] = fdiv((double)shared, (double)(Us > Ut ? Us : Ut));
  double d = md.bias;
#pragma unroll
  for (int k = 0; k < 6; ++k) d = fadd(d, fdiv(fmul(md.w[k], fsub(f[k], md.mean[k])), md.scale[k]));
  const double z = fadd(fmul(md.a, d), md.b);
  double p;
  if (z >= 0.0) {
    if (z < 700.0) {
      const double e = glibc_exp(-z, tab);
      p = fdiv(e, fadd(1.0, e));
    } else {
      p = 0.0;
    }
  } else {
    p = (z > -700.0) ? fdiv(1.0, fadd(1.0, glibc_exp(z, tab))) : 1.0;
  }
  if (0.0 > p) p = 0.0;
  if (1.0 < p) p = 1.0;
  return p;
}

__global__ void __launch_bounds__(kScoreThreads, 2) score_kernel(const ScoreArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ScoreSmem S;
  score_smem_layout(smem_raw, A.cap_u, A.cap_t, &S);

  const int64_t p = A.pair_ids ? A.pair_ids[blockIdx.x] : (int64_t)blockIdx.x;
  const int N = A.b.pair_n[p];
  const int M = A.b.pair_m[p];
  const int i0 = blockIdx.y * kScoreTile;
  const int jz0 = blockIdx.z * kScoreTile;
  if (i0 >= N || jz0 >= M) return;
  const int ni = min(kScoreTile, N - i0);
  const int jz1 = min(M, jz0 + kScoreTile);
  const int64_t s_first = A.b.pair_src[p] + i0;
  const int64_t t_first = A.b.pair_tgt[p];
  double *__restrict__ sim_out = A.sim + A.b.pair_sim_off[p];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int hbits = A.hash_bits;
  const int hslots = 1 << hbits;
  const TokenView tokens = A.b.tokens;
  const int64_t *__restrict__ row_ptr = A.d.row_ptr;
  const int32_t *__restrict__ dtgt = A.d.tgt;
  const double *__restrict__ dprob = A.d.prob;
  const int64_t n_rows = A.d.n_rows;

  for (int k = tid; k < 256; k += kScoreThreads) S.exp_tab[k] = kExpTableDev[k];
  for (int k = tid; k < ni; k += kScoreThreads) {
    S.src_off[k] = A.b.sent_tok_off[s_first + k];
    S.src_len[k] = A.b.sent_len[s_first + k];
    S.src_uniq[k] = A.b.sent_uniq[s_first + k];
    S.src_chars[k] = A.b.sent_chars[s_first + k];
  }

  for (int jc0 = jz0; jc0 < jz1;) {
    __syncthreads();  // previous chunk fully consumed
    if (tid == 0) {
      int su = 0, sl = 0, j = jc0;
      while (j < jz1) {
        const int u = A.b.sent_uniq[t_first + j], l = A.b.sent_len[t_first + j];
        if (u > A.cap_u || l > A.cap_t) {  // host pre-checks; never for valid launches
          atomicExch(A.status, BIMINE_E_LIMIT);
          break;
        }
        if (su + u > A.cap_u || sl + l > A.cap_t) break;
        su += u;
        sl += l;
        ++j;
      }
      S.misc[1] = j;
      S.misc[0] = 0;
    }
    __syncthreads();
    const int jc1 = S.misc[1];
    if (jc1 == jc0) return;  // capacity violation reported above
    const int nj = jc1 - jc0;
    if (tid < nj) {
      S.tgt_off[tid] = A.b.sent_tok_off[t_first + jc0 + tid];
      S.tgt_len[tid] = A.b.sent_len[t_first + jc0 + tid];
      S.tgt_uniq[tid] = A.b.sent_uniq[t_first + jc0 + tid];
      S.tgt_chars[tid] = A.b.sent_chars[t_first + jc0 + tid];
    }
    for (int k = tid; k < hslots; k += kScoreThreads) S.keys[k] = -1;
    for (int k = tid; k <= A.cap_t / 32; k += kScoreThreads) S.first[k] = 0u;
    __syncthreads();
    if (warp == 0) {  // exclusive prefix of occurrence counts over the chunk
      int run = 0;
      for (int base = 0; base < nj; base += 32) {
        const int j = base + lane;
        const int v = j < nj ? S.tgt_len[j] : 0;
        int x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(kFull, x, o);
          if (lane >= o) x += y;
        }
        if (j < nj) S.tgt_occ0[j] = run + x - v;
        run += __shfl_sync(kFull, x, 31);
      }
      if (lane == 0) S.tgt_occ0[nj] = run;
    }
    // ---- A1: insert the chunk's target tokens
    for (int jj = warp; jj < nj; jj += kScoreWarps) {
      const int64_t off = S.tgt_off[jj];
      const int L = S.tgt_len[jj];
      for (int k = lane; k < L; k += 32) hash_insert(S.keys, hbits, tokens[off + k]);
    }
    __syncthreads();
    // ---- A2: dense ids for occupied slots
    for (int k = tid; k < hslots; k += kScoreThreads) {
      if (S.keys[k] != -1) {
        const int d = atomicAdd(&S.misc[0], 1);
        S.dense[k] = (int16_t)d;
        S.colmask[d] = 0ull;
        S.reachcol[d] = 0ull;
        S.srccol[d] = 0ull;
      }
    }
    __syncthreads();
    // ---- A3: per occurrence: dense id, sentence membership, first flag
    for (int jj = warp; jj < nj; jj += kScoreWarps) {
      const int64_t off = S.tgt_off[jj];
      const int L = S.tgt_len[jj];
      const int q0 = S.tgt_occ0[jj];
      for (int k = lane; k < L; k += 32) {
        const int d = hash_find(S.keys, S.dense, hbits, tokens[off + k]);
        S.occ_d[q0 + k] = (int16_t)d;
        const unsigned long long old = atomicOr((unsigned long long *)&S.colmask[d], 1ull << jj);
        if (!((old >> jj) & 1ull)) atomicOr(&S.first[(q0 + k) >> 5], 1u << ((q0 + k) & 31));
      }
    }
    __syncthreads();
    // ---- B: source side -> srccol (shared tokens), reachcol (dictionary)
    for (int ii = warp; ii < ni; ii += kScoreWarps) {
      const int64_t off = S.src_off[ii];
      const int L = S.src_len[ii];
      const unsigned long long bit = 1ull << ii;
      for (int k = lane; k < L; k += 32) {
        const int32_t s = tokens[off + k];
        const int ds = hash_find(S.keys, S.dense, hbits, s);
        if (ds >= 0) atomicOr((unsigned long long *)&S.srccol[ds], bit);
        if (s >= 0 && s < n_rows) {
          const int64_t e1 = row_ptr[s + 1];
          for (int64_t e = row_ptr[s]; e < e1; ++e) {
            const int d = hash_find(S.keys, S.dense, hbits, dtgt[e]);
            if (d >= 0) atomicOr((unsigned long long *)&S.reachcol[d], bit);
          }
        }
      }
    }
    __syncthreads();
    // ---- C: covered_target and shared counts, lanes over source sentences
    for (int jj = warp; jj < nj; jj += kScoreWarps) {
      const int q0 = S.tgt_occ0[jj];
      const int L = S.tgt_len[jj];
      uint32_t lo = 0, hi = 0;
      for (int k = 0; k < L; ++k) {
        const int q = q0 + k;
        const int d = S.occ_d[q];
        const uint64_t r = S.reachcol[d];
        lo += (uint32_t)(r >> lane) & 1u;
        hi += (uint32_t)(r >> (lane + 32)) & 1u;
        if ((S.first[q >> 5] >> (q & 31)) & 1u) {
          const uint64_t sc = S.srccol[d];
          lo += ((uint32_t)(sc >> lane) & 1u) << 16;
          hi += ((uint32_t)(sc >> (lane + 32)) & 1u) << 16;
        }
      }
      S.cnt[lane * kCntStride + jj] = lo;
      S.cnt[(lane + 32) * kCntStride + jj] = hi;
    }
    __syncthreads();
    // ---- D: per source sentence, lanes over target sentences
    uint64_t *rany = S.rec_any + warp * 32;
    uint64_t *rm = S.rec_m + warp * 32 * kCandInline;
    double *rp = S.rec_p + warp * 32 * kCandInline;
    int32_t *rs = S.rec_s + warp * 32;
    uint8_t *rnc = S.rec_nc + warp * 32;
    const int jlo = lane, jhi = lane + 32;
    for (int ii = warp; ii < ni; ii += kScoreWarps) {
      const int64_t off = S.src_off[ii];
      const int L = S.src_len[ii];
      int cov_lo = 0, cov_hi = 0;
      double sum_lo = 0.0, sum_hi = 0.0;
      for (int seg = 0; seg < L; seg += 32) {
        const int k = seg + lane;
        uint64_t any = 0ull;
        int nc = 0;
        int32_t s = -1;
        if (k < L) {
          s = tokens[off + k];
          if (s >= 0 && s < n_rows) {
            const int64_t e1 = row_ptr[s + 1];
            for (int64_t e = row_ptr[s]; e < e1; ++e) {
              const int d = hash_find(S.keys, S.dense, hbits, dtgt[e]);
              if (d >= 0) {
                const uint64_t m = S.colmask[d];
                any |= m;
                if (nc < kCandInline) {
                  rm[lane * kCandInline + nc] = m;
                  rp[lane * kCandInline + nc] = dprob[e];
                }
                ++nc;
              }
            }
          }
        }
        rany[lane] = any;
        rnc[lane] = (uint8_t)(nc > kCandInline ? 255 : nc);
        rs[lane] = s;
        __syncwarp();
        const int kn = min(32, L - seg);
        for (int kk = 0; kk < kn; ++kk) {
          const uint64_t ah = rany[kk];
          if (ah == 0ull) continue;
          const bool hl = (ah >> jlo) & 1ull;
          const bool hh = (ah >> jhi) & 1ull;
          if (!(hl | hh)) continue;
          double bl = 0.0, bh = 0.0;
          const int c = rnc[kk];
          if (c != 255) {
            for (int cc = 0; cc < c; ++cc) {
              const uint64_t m = rm[kk * kCandInline + cc];
              const double pr = rp[kk * kCandInline + cc];
              if (((m >> jlo) & 1ull) && pr > bl) bl = pr;
              if (((m >> jhi) & 1ull) && pr > bh) bh = pr;
            }
          } else {  // long dictionary row: walk it again from global memory
            const int32_t sk = rs[kk];
            const int64_t e1 = row_ptr[sk + 1];
            for (int64_t e = row_ptr[sk]; e < e1; ++e) {
              const int d = hash_find(S.keys, S.dense, hbits, dtgt[e]);
              if (d >= 0) {
                const uint64_t m = S.colmask[d];
                const double pr = dprob[e];
                if (((m >> jlo) & 1ull) && pr > bl) bl = pr;
                if (((m >> jhi) & 1ull) && pr > bh) bh = pr;
              }
            }
          }
          if (hl) {
            ++cov_lo;
            sum_lo = fadd(sum_lo, bl);
          }
          if (hh) {
            ++cov_hi;
            sum_hi = fadd(sum_hi, bh);
          }
        }
        __syncwarp();
      }
      const int Ls = L, Us = S.src_uniq[ii], Cs = S.src_chars[ii];
      double *row = sim_out + (int64_t)(i0 + ii) * M + jc0;
      if (jlo < nj) {
        const uint32_t c = S.cnt[ii * kCntStride + jlo];
        row[jlo] = cell_score(A.md, Ls, Us, Cs, S.tgt_len[jlo], S.tgt_uniq[jlo], S.tgt_chars[jlo], cov_lo, sum_lo,
                              (int)(c & 0xffffu), (int)(c >> 16), S.exp_tab);
      }
      if (jhi < nj) {
        const uint32_t c = S.cnt[ii * kCntStride + jhi];
        row[jhi] = cell_score(A.md, Ls, Us, Cs, S.tgt_len[jhi], S.tgt_uniq[jhi], S.tgt_chars[jhi], cov_hi, sum_hi,
                              (int)(c & 0xffffu), (int)(c >> 16), S.exp_tab);
      }
    }
    jc0 = jc1;
  }
}

}  // namespace bimine
