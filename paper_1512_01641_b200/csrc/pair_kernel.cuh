// pair_kernel.cuh -- score matrix of one document pair per CTA.
//
// build_score_matrix (align.py:102-129) for pairs with N, M <= 64 and
// sentences of <= 255 tokens (all C2/C4/C5 pairs); larger pairs (C1, C3)
// run the same kernel over 64x64 sentence tiles, (pair, i0, j0) per CTA.
// 8 warps, 4 CTAs per SM; the per-pair tables live in shared memory, the
// per-cell counters in global scratch (L2-resident while the CTA works).
//
//  A  target hash: every target token of the chunk -> dense id d;
//     colmask[d] = 64-bit set of target sentences containing d.
//  D  warp per source sentence i (claimed longest first); lane j owns
//     target sentences j and j + 32.  The sentence's occurrences are cut
//     into segments of <= 32 occurrences whose dictionary rows (p > 0
//     entries, CSR) total <= 96 entries.  The warp walks a segment's
//     entries flattened, 32 per step, against the hash (behind a Bloom
//     prefilter); each hit (colmask, p) is appended to the warp's
//     candidate list in entry order and sets reachcol[d] |= bit i
//     (reachable_targets, classifier.py:54-59).  Then, occurrence by
//     occurrence in order, lane j takes the max p over the occurrence's
//     candidates present in sentence j and adds it to the running sum --
//     the exact sequential sum of classifier.py:75-82 -- and counts it in
//     `covered` when > 0 (all p > 0).  Shared tokens (classifier.py:94):
//     the first occurrence of each distinct chunk token (a per-warp seen
//     bitmap) adds its colmask bits.
//  C  warp per target sentence j, lanes = occurrences: transposing the
//     reachcol rows gives covered_target(i, j) by popc
//     (classifier.py:88-92), multiplicities included.
//  F  all threads, one cell each (flattened, full lanes): six features ->
//     margin -> logistic (terms.cuh), one coalesced store per cell.  The
//     running sums of D are parked in the cell's own output slot (L2) and
//     overwritten here.
//
// If the chunk's distinct target tokens exceed the hash capacity the
// target side is processed in halves (same results, more passes).
#pragma once

#include "common.cuh"
#include "nw_kernel.cuh"
#include "terms.cuh"

namespace bimine {

constexpr int kPairThreads = 256;
constexpr int kPairWarps = kPairThreads / 32;
constexpr int kPairMax = 64;         // sentences per side
constexpr int kPairMaxLen = 255;     // tokens per sentence (u8 counts)
constexpr int kCellStride = 64;      // per-cell arrays are [64][64]

struct PairArgs {
  BatchDev b;
  DictDev d;
  Model md;
  TermTables T;
  double *sim;
  uint16_t *aux;            // per-cell scratch, same layout as sim: covered | shared << 8
  const int64_t *tiles;     // (pair, i0, j0) per tile of the pairs larger than 64x64
  int64_t n_tiles;          // CTAs [0, n_tiles) are tiles, the rest one pair each
  int cap_u;                // distinct target tokens per chunk (dense arrays)
  int hash_bits;            // log2(hash slots) >= log2(2 cap_u)
  int cap_t;                // target occurrences per chunk
  // fused NW + traceback + filter for one-CTA pairs (null: score only)
  bimine_match *nw_matches;  // slots at nw_out_off[pair]
  const int64_t *nw_out_off;
  int32_t *nw_counts;
  double *nw_score;          // optional
  double gap, threshold, mismatch, bonus;
  // features mode (extract_features, classifier.py:62-112): the six
  // features of every cell at features[6 * (pair_sim_off + i * M + j) + k]
  double *features;
  // upload gate (bimine_mine_host): pair p's data are on the device once
  // *ready >= need[p] (the counter grows as pieces land); null: no wait
  const int32_t *ready;
  const int32_t *need;
};

constexpr int kSegItems = 96;   // dictionary entries examined per warp segment
constexpr int kBloomBits = 14;  // 16384-bit prefilter in front of the hash

struct PairSmem {
  uint64_t *colmask;   // [cap_u]
  uint64_t *reachcol;  // [cap_u]
  uint64_t *c_m;       // [warps][kSegItems] in-chunk translations: colmask
  double *c_p;         // [warps][kSegItems]                        probability (negated: first of its occurrence)
  int64_t *src_off, *tgt_off;  // [64]
  uint32_t *bloom;     // [2^kBloomBits / 32]
  int32_t *keys;       // [slots]
  int32_t *src_len, *src_uniq, *src_chars;  // [64]
  int32_t *tgt_len, *tgt_uniq, *tgt_chars;  // [64]
  int32_t *tgt_occ0;   // [65] chunk-local occurrence offsets
  uint8_t *src_order;  // [64] source sentences, longest first (phase D claim order)
  uint32_t *seen;      // [warps][1024 / 32] chunk tokens already met in the warp's source sentence
  int32_t *misc;       // [8]: 0 distinct count, 1 chunk end, 2 D work counter, 3 C work counter
  int16_t *dense;      // [slots]
  int16_t *tgt_d;      // [cap_t]
  uint8_t *covt;       // [64][64]
  size_t overlay_bytes;  // bytes of the reusable region at the start
};

// fused-NW scratch inside the overlay: sim tile [64][64] f64, row buffer, directions
constexpr size_t kNwTileBytes = 64 * 64 * 8;
constexpr size_t kNwRowBytes = 66 * 8;
constexpr size_t kNwDirBytes = 65 * 5 * 4;

__host__ __device__ inline size_t pair_smem_layout(unsigned char *base, int cap_u, int hash_bits, int cap_t,
                                                   PairSmem *s) {
  size_t o = 0;
  auto take = [&](size_t bytes, size_t al) -> unsigned char * {
    o = (o + al - 1) / al * al;
    unsigned char *p = base ? base + o : nullptr;
    o += bytes;
    return p;
  };
  const size_t slots = (size_t)1 << hash_bits;
  PairSmem t;
  // region reused by the fused NW once the score phases are done
  t.colmask = (uint64_t *)take((size_t)cap_u * 8, 16);
  t.reachcol = (uint64_t *)take((size_t)cap_u * 8, 16);
  t.c_m = (uint64_t *)take((size_t)kPairWarps * kSegItems * 8, 16);
  t.c_p = (double *)take((size_t)kPairWarps * kSegItems * 8, 16);
  t.bloom = (uint32_t *)take(((size_t)1 << kBloomBits) / 8, 16);
  t.keys = (int32_t *)take(slots * 4, 16);
  t.dense = (int16_t *)take(slots * 2, 4);
  t.tgt_d = (int16_t *)take((size_t)cap_t * 2, 4);
  t.seen = (uint32_t *)take((size_t)kPairWarps * 32 * 4, 16);
  t.overlay_bytes = o;
  // live until the end
  t.src_off = (int64_t *)take(64 * 8, 16);
  t.tgt_off = (int64_t *)take(64 * 8, 16);
  t.src_len = (int32_t *)take(64 * 4, 4);
  t.src_uniq = (int32_t *)take(64 * 4, 4);
  t.src_chars = (int32_t *)take(64 * 4, 4);
  t.tgt_len = (int32_t *)take(64 * 4, 4);
  t.tgt_uniq = (int32_t *)take(64 * 4, 4);
  t.tgt_chars = (int32_t *)take(64 * 4, 4);
  t.tgt_occ0 = (int32_t *)take(65 * 4, 4);
  t.misc = (int32_t *)take(8 * 4, 4);
  t.src_order = (uint8_t *)take(64, 4);
  t.covt = (uint8_t *)take(64 * 64, 4);
  if (s) *s = t;
  return (o + 15) / 16 * 16;
}

// lane j of the result holds bit k = bit j of lane k's x (32x32 bit transpose)
__device__ __forceinline__ uint32_t transpose32(uint32_t x, int lane) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const uint32_t m = (s == 16) ? 0x0000FFFFu : (s == 8) ? 0x00FF00FFu : (s == 4) ? 0x0F0F0F0Fu
                       : (s == 2) ? 0x33333333u : 0x55555555u;
    const uint32_t o = __shfl_xor_sync(kFull, x, s);
    // lower lane: keep x & m, take (o & m) << s; upper lane: keep x & ~m,
    // take (o & ~m) >> s -- one bit-select with the lane's keep mask
    const bool up = (lane & s) != 0;
    const uint32_t keep = up ? ~m : m;
    const uint32_t v = up ? (o >> s) : (o << s);
    x = (x & keep) | (v & ~keep);
  }
  return x;
}

__device__ __forceinline__ uint32_t bloom_bit(int32_t key) {
  return ((uint32_t)key * 0x85EBCA6Bu) >> (32 - kBloomBits);
}

__device__ __forceinline__ int pk_find(const int32_t *keys, const int16_t *dense, int bits, int32_t key) {
  const uint32_t mask = (1u << bits) - 1u;
  uint32_t slot = hash_slot(key, 32 - bits);
  while (true) {
    const int32_t k = keys[slot];
    if (k == key) return dense[slot];
    if (k == -1) return -1;
    slot = (slot + 1u) & mask;
  }
}

// lookup behind the Bloom prefilter (most dictionary translations are absent)
__device__ __forceinline__ int pk_find_f(const uint32_t *bloom, const int32_t *keys, const int16_t *dense, int bits,
                                         int32_t key) {
  const uint32_t b = bloom_bit(key);
  if (!((bloom[b >> 5] >> (b & 31)) & 1u)) return -1;
  return pk_find(keys, dense, bits, key);
}

__device__ __forceinline__ void pk_insert(int32_t *keys, int bits, int32_t key) {
  const uint32_t mask = (1u << bits) - 1u;
  uint32_t slot = hash_slot(key, 32 - bits);
  while (true) {
    const int32_t k = keys[slot];
    if (k == key) return;
    if (k == -1) {
      const int32_t prev = atomicCAS(&keys[slot], -1, key);
      if (prev == -1 || prev == key) return;
    }
    slot = (slot + 1u) & mask;
  }
}

// (bit != 0 && p > best) ? p : best, as one predicate: the bit test feeds
// the compare's predicate input (LOP3 + DSETP.AND + two selects; written
// in C++ the compiler selects twice, four FSELs per half)
__device__ __forceinline__ double max_if_bit(double best, double p, uint32_t bit) {
  double r;
  asm("{\n\t.reg .pred q;\n\t"
      "setp.ne.u32 q, %3, 0;\n\t"
      "setp.gt.and.f64 q, %2, %1, q;\n\t"
      "selp.f64 %0, %2, %1, q;\n\t}"
      : "=d"(r)
      : "d"(best), "d"(p), "r"(bit));
  return r;
}

// 64-bit OR into shared memory as native 32-bit ORs of the nonzero halves
// (a 64-bit shared atomicOr compiles to a compare-and-swap loop)
__device__ __forceinline__ void or64(uint64_t *w, uint64_t m) {
  uint32_t *h = (uint32_t *)w;
  if ((uint32_t)m) atomicOr(h, (uint32_t)m);
  if ((uint32_t)(m >> 32)) atomicOr(h + 1, (uint32_t)(m >> 32));
}

// Is the pair handled by pair_kernel?  (host and device agree on this rule)
__host__ __device__ inline bool pair_is_small(int n, int m, int max_len) {
  return n <= kPairMax && m <= kPairMax && max_len <= kPairMaxLen;
}

// kFeatures: also write the six features per cell (bimine_features_batch)
template <bool kFeatures>
__global__ void __launch_bounds__(kPairThreads, 4) pair_kernel(const PairArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // CTAs [0, n_tiles) take the 64x64 tiles of large pairs (first, so the
  // long pairs start early), the rest one pair each (pairs larger than
  // 64x64 are skipped there: their tiles cover them)
  int64_t p;
  int i0 = 0, j0 = 0;
  const bool is_tile = (int64_t)blockIdx.x < A.n_tiles;
  if (is_tile) {
    p = A.tiles[3 * (int64_t)blockIdx.x];
    i0 = (int)A.tiles[3 * (int64_t)blockIdx.x + 1];
    j0 = (int)A.tiles[3 * (int64_t)blockIdx.x + 2];
  } else {
    p = (int64_t)blockIdx.x - A.n_tiles;
  }
  if (A.ready) {  // wait until the chunk holding this pair's data has landed
    if (threadIdx.x == 0) {
      const int want = A.need[p];
      while (true) {
        int r;
        asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(r) : "l"(A.ready) : "memory");
        if (r >= want) break;
        __nanosleep(256);
      }
    }
    __syncthreads();
  }
  const int Nfull = A.b.pair_n[p], Mfull = A.b.pair_m[p];
  if (!is_tile && (Nfull > kPairMax || Mfull > kPairMax)) return;
  // this CTA's block: source sentences [i0, i0 + N), target sentences [j0, j0 + M)
  const int N = min(kPairMax, Nfull - i0), M = min(kPairMax, Mfull - j0);
  PairSmem S;
  const int hbits = A.hash_bits;
  pair_smem_layout(smem_raw, A.cap_u, hbits, A.cap_t, &S);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t s_first = A.b.pair_src[p] + i0, t_first = A.b.pair_tgt[p] + j0;
  const int32_t *__restrict__ tokens = A.b.tokens;
  const int64_t *__restrict__ row_ptr = A.d.row_ptr;
  const int32_t *__restrict__ dtgt = A.d.tgt;
  const double *__restrict__ dprob = A.d.prob;
  const int64_t n_rows = A.d.n_rows;
  const int hslots = 1 << hbits;
  // the block's cell (i, j) lives at out[i * Mfull + j]; also the running-sum scratch
  double *__restrict__ out = A.sim + A.b.pair_sim_off[p] + (int64_t)i0 * Mfull + j0;
  uint16_t *__restrict__ aux = A.aux + A.b.pair_sim_off[p] + (int64_t)i0 * Mfull + j0;

  // ---- 0: tables and sentence metadata
  if (tid < N) {
    S.src_off[tid] = A.b.sent_tok_off[s_first + tid];
    S.src_len[tid] = A.b.sent_len[s_first + tid];
    S.src_uniq[tid] = A.b.sent_uniq[s_first + tid];
    S.src_chars[tid] = A.b.sent_chars[s_first + tid];
  } else if (tid >= 64 && tid - 64 < M) {
    const int j = tid - 64;
    S.tgt_off[j] = A.b.sent_tok_off[t_first + j];
    S.tgt_len[j] = A.b.sent_len[t_first + j];
    S.tgt_uniq[j] = A.b.sent_uniq[t_first + j];
    S.tgt_chars[j] = A.b.sent_chars[t_first + j];
  }
  __syncthreads();
  {  // the rule of pair_is_small: every sentence <= kPairMaxLen tokens
    const int l = tid < N ? S.src_len[tid] : (tid >= 64 && tid - 64 < M) ? S.tgt_len[tid - 64] : 0;
    if (__syncthreads_or(l > kPairMaxLen)) return;
  }
  if (tid < N) {  // phase D claims source sentences longest first (shorter tail at its barrier)
    const int li = S.src_len[tid];
    int rank = 0;
    for (int k = 0; k < N; ++k) {
      const int lk = S.src_len[k];
      rank += (lk > li) || (lk == li && k < tid);
    }
    S.src_order[rank] = (uint8_t)tid;
  }
  __syncthreads();

  for (int jc0 = 0; jc0 < M;) {
    // ---- chunk [jc0, jc1): at most cap_t target occurrences
    if (warp == 0) {
      int run = 0, end = jc0;
      for (int base = jc0; base < M; base += 32) {
        const int j = base + lane;
        const int v = j < M ? S.tgt_len[j] : 0;
        int x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(kFull, x, o);
          if (lane >= o) x += y;
        }
        const unsigned ok = __ballot_sync(kFull, j < M && run + x <= A.cap_t);
        const int cnt = __popc(ok);  // lengths >= 0: the fitting lanes are a prefix
        end = base + cnt;
        if (cnt < 32) break;
        run += __shfl_sync(kFull, x, 31);
      }
      if (lane == 0) S.misc[1] = max(end, jc0 + 1);
    }
    __syncthreads();
    int jc1 = S.misc[1];
    while (true) {
      const int nj = jc1 - jc0;
      if (warp == 0) {  // chunk-local occurrence offsets
        int run = 0;
        for (int base = 0; base < nj; base += 32) {
          const int jj = base + lane;
          const int v = jj < nj ? S.tgt_len[jc0 + jj] : 0;
          int x = v;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(kFull, x, o);
            if (lane >= o) x += y;
          }
          if (jj < nj) S.tgt_occ0[jj] = run + x - v;
          run += __shfl_sync(kFull, x, 31);
        }
        if (lane == 0) {
          S.tgt_occ0[nj] = run;
          S.misc[0] = 0;
          S.misc[2] = 0;
          S.misc[3] = 0;
        }
      }
      for (int k = tid; k < hslots; k += kPairThreads) S.keys[k] = -1;
      for (int k = tid; k < (1 << kBloomBits) / 32; k += kPairThreads) S.bloom[k] = 0u;
      __syncthreads();
      // ---- A1: insert the chunk's target tokens (+ prefilter bits)
      for (int jj = warp; jj < nj; jj += kPairWarps) {
        const int64_t off = S.tgt_off[jc0 + jj];
        const int L = S.tgt_len[jc0 + jj];
        for (int k = lane; k < L; k += 32) {
          const int32_t t = tokens[off + k];
          pk_insert(S.keys, hbits, t);
          const uint32_t b = bloom_bit(t);
          atomicOr(&S.bloom[b >> 5], 1u << (b & 31));
        }
      }
      __syncthreads();
      // ---- A2: dense ids
      for (int k = tid; k < hslots; k += kPairThreads) {
        if (S.keys[k] != -1) {
          const int d = atomicAdd(&S.misc[0], 1);
          if (d < A.cap_u) {
            S.dense[k] = (int16_t)d;
            S.colmask[d] = 0ull;
            S.reachcol[d] = 0ull;
          }
        }
      }
      __syncthreads();
      if (S.misc[0] <= A.cap_u || nj == 1) break;
      jc1 = jc0 + nj / 2;  // too many distinct tokens: halve the chunk
      __syncthreads();
    }
    const int nj = jc1 - jc0;
    // ---- A3: occurrences -> dense id, sentence sets
    for (int jj = warp; jj < nj; jj += kPairWarps) {
      const int64_t off = S.tgt_off[jc0 + jj];
      const int L = S.tgt_len[jc0 + jj];
      const int q0 = S.tgt_occ0[jj];
      for (int k = lane; k < L; k += 32) {
        const int d = pk_find(S.keys, S.dense, hbits, tokens[off + k]);
        S.tgt_d[q0 + k] = (int16_t)d;
        or64(&S.colmask[d], 1ull << jj);
      }
    }
    __syncthreads();
    // ---- D: source side, warps take sentences dynamically
    {
      // phase D's lane id, read once (%laneid) and opaque to ptxas like
      // cbase below, so that it is not re-derived from %tid per segment
      int lane_r;
      asm volatile("mov.u32 %0, %%laneid;" : "=r"(lane_r));
      const int lane = lane_r;
      // the warp's candidate-list offset, opaque to ptxas so that it stays
      // in a register rather than being re-derived from %tid in the loops
      int cbase;
      asm volatile("mov.u32 %0, %1;" : "=r"(cbase) : "r"(warp * kSegItems));
      uint64_t *cm = S.c_m + cbase;
      uint32_t *seen = S.seen + warp * 32;
      double *cp = S.c_p + cbase;
      const int jlo = lane, jhi = lane + 32;
      const unsigned lt_mask = (1u << lane) - 1u;
      // software pipeline: the next segment's window (token, dictionary row)
      // is loaded while the current one is processed, and the next
      // sentence is claimed one sentence ahead
      auto claim = [&]() -> int {
        int v = 0;
        if (lane == 0) {
          v = atomicAdd(&S.misc[2], 1);
          v = v < N ? (int)S.src_order[v] : N;
        }
        return __shfl_sync(kFull, v, 0);
      };
      auto load_tok = [&](int si, int pos) -> int32_t {
        if (si >= N) return -1;
        const int k = pos + lane;
        return k < S.src_len[si] ? tokens[S.src_off[si] + k] : -1;
      };
      int i = claim();
      int i_nxt = i < N ? claim() : N;
      int32_t s_w = load_tok(i, 0);
      int64_t e0_w = 0;
      int rl_w = 0;
      if (s_w >= 0 && s_w < n_rows) {
        e0_w = row_ptr[s_w];
        rl_w = (int)(row_ptr[s_w + 1] - e0_w);
      }
      while (i < N) {
        const int L = S.src_len[i];
        const unsigned long long ibit = 1ull << i;
        int cov_lo = 0, cov_hi = 0, sh_lo = 0, sh_hi = 0;
        double sum_lo = 0.0, sum_hi = 0.0;
        seen[lane] = 0u;  // (cap_u = 1024 dense ids: 32 words)
        __syncwarp();
        for (int seg = 0; seg < L;) {
          const int k = seg + lane;
          const bool valid = k < L;
          const int32_t s = s_w;  // token k of sentence i, or -1
          const int64_t e0 = e0_w;
          const int rl = rl_w;
          // segment: the longest prefix of occurrences whose rows total
          // <= kSegItems entries (at least one occurrence)
          int x = rl;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(kFull, x, o);
            if (lane >= o) x += y;
          }
          const unsigned fitm = __ballot_sync(kFull, valid && (x <= kSegItems || lane == 0));
          const int cnt = __popc(fitm);
          const bool in_seg = lane < cnt;
          const int items = min(kSegItems, __shfl_sync(kFull, x, cnt - 1));
          const int ofs = x - rl;  // exclusive prefix: first item of this occurrence
          const int64_t eb = e0 - ofs;  // entry of item `it` of this occurrence: eb + it (one 64-bit shuffle)
          // the segment's dictionary entries (<= 3 steps of 32, in order):
          // the first two steps' owners found and loads issued now, so their
          // L2 latency overlaps the shared-token work below
          static_assert(kSegItems == 96, "the walk below is three steps");
          int w_owner[2];
          int32_t w_tgt[2];
          double w_p[2];
#pragma unroll
          for (int st = 0; st < 2; ++st) {
            w_owner[st] = 0;
            w_tgt[st] = -1;
            w_p[st] = 0.0;
            if (st * 32 < items) {  // warp-uniform
              const int it = st * 32 + lane;
              int owner = 0;  // last segment lane whose first item <= it
#pragma unroll
              for (int step = 16; step >= 1; step >>= 1) {
                const int cand = owner + step;
                const int v = __shfl_sync(kFull, ofs, cand & 31);
                // (no cand < cnt test: ofs is the exclusive prefix, so every
                // lane from cnt on has ofs >= x[cnt - 1] >= items > it)
                if (v <= it) owner = cand;
              }
              const int64_t oeb = __shfl_sync(kFull, eb, owner);
              w_owner[st] = owner;
              if (it < items) {
                const int64_t e = oeb + it;
                w_tgt[st] = dtgt[e];
                w_p[st] = dprob[e];
              }
            }
          }
          // next window: the rest of this sentence, else the next sentence
          const bool more = seg + cnt < L;
          const int32_t tok_nx = more ? load_tok(i, seg + cnt) : load_tok(i_nxt, 0);
          // shared tokens: first occurrence of a source token that is a chunk
          // token (one lane of each distinct dense id claims its seen bit)
          const int ds = in_seg ? pk_find_f(S.bloom, S.keys, S.dense, hbits, s) : -1;
          bool first = false;
          if (ds >= 0) {
            const uint32_t bit = 1u << (ds & 31);
            first = !(atomicOr(&seen[ds >> 5], bit) & bit);
          }
          const uint64_t shm = first ? S.colmask[ds] : 0ull;
          for (unsigned sb = __ballot_sync(kFull, shm != 0ull); sb; sb &= sb - 1u) {
            const uint64_t mm = __shfl_sync(kFull, shm, __ffs(sb) - 1);
            sh_lo += (int)(((uint32_t)mm >> lane) & 1u);
            sh_hi += (int)(((uint32_t)(mm >> 32) >> lane) & 1u);
          }
          const int rl0 = __shfl_sync(kFull, rl, 0);
          if (rl0 > kSegItems) {
            // a lone occurrence whose row exceeds the segment (cnt == 1): the
            // whole warp walks the row and reduces the per-sentence maxima
            const int64_t r0 = __shfl_sync(kFull, e0, 0);
            uint64_t a = 0ull;
            double bl = 0.0, bh = 0.0;
            for (int base = 0; base < rl0; base += 32) {
              const int it = base + lane;
              int d = -1;
              if (it < rl0) d = pk_find_f(S.bloom, S.keys, S.dense, hbits, dtgt[r0 + it]);
              const uint64_t m = d >= 0 ? S.colmask[d] : 0ull;
              const double pr = d >= 0 ? dprob[r0 + it] : 0.0;
              if (d >= 0) or64(&S.reachcol[d], ibit);
              unsigned bal = __ballot_sync(kFull, d >= 0);
              while (bal) {
                const int src = __ffs(bal) - 1;
                bal &= bal - 1u;
                const uint64_t mm = __shfl_sync(kFull, m, src);
                const double pp = __shfl_sync(kFull, pr, src);
                a |= mm;
                if (((mm >> jlo) & 1ull) && pp > bl) bl = pp;
                if (((mm >> jhi) & 1ull) && pp > bh) bh = pp;
              }
            }
            if (a != 0ull) {
              sum_lo = fadd(sum_lo, bl);
              sum_hi = fadd(sum_hi, bh);
              cov_lo += (int)((a >> jlo) & 1ull);
              cov_hi += (int)((a >> jhi) & 1ull);
            }
            s_w = tok_nx;
            e0_w = 0;
            rl_w = 0;
            if (s_w >= 0 && s_w < n_rows) {
              e0_w = row_ptr[s_w];
              rl_w = (int)(row_ptr[s_w + 1] - e0_w);
            }
            seg += 1;  // cnt == 1 here
            continue;
          }
          // all dictionary entries of the segment, 32 at a time, in order.
          // A candidate whose owner differs from the previous candidate's
          // (the first of its occurrence) is stored with p negated: every
          // dictionary p is > 0, so the sign bit is free and the pass below
          // needs no owner array
          int ncand = 0;
          int last_owner = -1;  // owner of the segment's latest candidate
#pragma unroll
          for (int st = 0; st < 3; ++st) {
            if (st * 32 >= items) break;  // warp-uniform
            int owner;
            double pr;
            int32_t tg;
            if (st < 2) {
              owner = w_owner[st];
              pr = w_p[st];  // loaded with the id: no second round trip for hits
              tg = w_tgt[st];
            } else {
              const int it = 64 + lane;
              owner = 0;
#pragma unroll
              for (int step = 16; step >= 1; step >>= 1) {
                const int cand = owner + step;
                const int v = __shfl_sync(kFull, ofs, cand & 31);
                if (v <= it) owner = cand;
              }
              const int64_t oeb = __shfl_sync(kFull, eb, owner);
              tg = -1;
              pr = 0.0;
              if (it < items) {
                const int64_t e = oeb + it;
                tg = dtgt[e];
                pr = dprob[e];
              }
            }
            const int d = tg >= 0 ? pk_find_f(S.bloom, S.keys, S.dense, hbits, tg) : -1;
            const bool pres = d >= 0;
            const unsigned bal = __ballot_sync(kFull, pres);
            const unsigned below = bal & lt_mask;
            const int prev_sh = __shfl_sync(kFull, owner, below ? 31 - __clz(below) : 0);
            if (pres) {
              const uint64_t m = S.colmask[d];
              const int pos = ncand + __popc(below);
              const int prev = below ? prev_sh : last_owner;
              cm[pos] = m;
              cp[pos] = owner != prev ? -pr : pr;
              or64(&S.reachcol[d], ibit);
            }
            if (bal) last_owner = __shfl_sync(kFull, owner, 31 - __clz(bal));
            ncand += __popc(bal);
          }
          // the next window's dictionary rows (its tokens arrived during the walk)
          s_w = tok_nx;
          e0_w = 0;
          rl_w = 0;
          if (s_w >= 0 && s_w < n_rows) {
            e0_w = row_ptr[s_w];
            rl_w = (int)(row_ptr[s_w + 1] - e0_w);
          }
          __syncwarp();
          // occurrence-major, in order: max p over the occurrence's
          // translations present in sentence j, added to the running sum
          // (adding +0.0 when absent leaves the non-negative sum unchanged)
          // bit of target jlo in the low word, jhi in the high word; read once
          // per segment through volatile asm so that ptxas keeps it in a
          // register instead of re-deriving it from %tid in the loop
          uint32_t lbit;
          asm volatile("mov.u32 %0, %%lanemask_eq;" : "=r"(lbit));
          // candidate-major: the candidates are in entry order, so each
          // occurrence's are contiguous and the occurrences come in order;
          // an occurrence's best is added when the next one starts (a
          // negated p) or the list ends.  The flush before the first
          // candidate adds +0.0 to a non-negative sum: bit-identical
          // (occurrences without a candidate would add +0.0 too)
          double bl = 0.0, bh = 0.0;
          for (int c = 0; c < ncand; ++c) {
            const uint64_t m = cm[c];  // same address in every lane: broadcast
            double pr = cp[c];
            if (pr < 0.0) {  // warp-uniform
              // every dictionary probability is > 0, so a translation of
              // the occurrence is in sentence j exactly when its best > 0
              sum_lo = fadd(sum_lo, bl);
              sum_hi = fadd(sum_hi, bh);
              cov_lo += bl > 0.0 ? 1 : 0;
              cov_hi += bh > 0.0 ? 1 : 0;
              bl = 0.0;
              bh = 0.0;
              pr = -pr;
            }
            bl = max_if_bit(bl, pr, (uint32_t)m & lbit);
            bh = max_if_bit(bh, pr, (uint32_t)(m >> 32) & lbit);
          }
          if (ncand > 0) {
            sum_lo = fadd(sum_lo, bl);
            sum_hi = fadd(sum_hi, bh);
            cov_lo += bl > 0.0 ? 1 : 0;
            cov_hi += bh > 0.0 ? 1 : 0;
          }
          __syncwarp();
          seg += cnt;
        }
        if (jlo < nj) {
          aux[(int64_t)i * Mfull + jc0 + jlo] = (uint16_t)(cov_lo | (sh_lo << 8));
          out[(int64_t)i * Mfull + jc0 + jlo] = sum_lo;
        }
        if (jhi < nj) {
          aux[(int64_t)i * Mfull + jc0 + jhi] = (uint16_t)(cov_hi | (sh_hi << 8));
          out[(int64_t)i * Mfull + jc0 + jhi] = sum_hi;
        }
        if (L == 0) {  // (the builder rejects empty sentences; keep the pipeline consistent anyway)
          s_w = load_tok(i_nxt, 0);
          e0_w = 0;
          rl_w = 0;
          if (s_w >= 0 && s_w < n_rows) {
            e0_w = row_ptr[s_w];
            rl_w = (int)(row_ptr[s_w + 1] - e0_w);
          }
        }
        i = i_nxt;  // its first window is already loaded
        if (i < N) i_nxt = claim();
      }
    }
    __syncthreads();
    // ---- C: covered_target, warps take target sentences, lanes over occurrences
    while (true) {
      int jj = 0;
      if (lane == 0) jj = atomicAdd(&S.misc[3], 1);
      jj = __shfl_sync(kFull, jj, 0);
      if (jj >= nj) break;
      const int q0 = S.tgt_occ0[jj];
      const int L = S.tgt_len[jc0 + jj];
      int c_lo = 0, c_hi = 0;
      for (int seg = 0; seg < L; seg += 32) {
        const uint64_t r = (seg + lane < L) ? S.reachcol[S.tgt_d[q0 + seg + lane]] : 0ull;
        c_lo += __popc(transpose32((uint32_t)r, lane));
        c_hi += __popc(transpose32((uint32_t)(r >> 32), lane));
      }
      if (lane < N) S.covt[lane * kCellStride + jc0 + jj] = (uint8_t)c_lo;
      if (lane + 32 < N) S.covt[(lane + 32) * kCellStride + jc0 + jj] = (uint8_t)c_hi;
    }
    jc0 = jc1;
    __syncthreads();
  }

  // ---- F: finalize, one cell per thread, coalesced loads/stores
  const bool fuse_nw = A.nw_matches != nullptr && !is_tile;
  double *tile = (double *)smem_raw;  // overlay: dead after phase C
  const int cells = N * M;
  // cell c = i * M + j, stepped without integer division
  const int di = kPairThreads / M, dj = kPairThreads - di * M;
  int i = tid / M, j = tid - (tid / M) * M;
  for (int c = tid; c < cells; c += kPairThreads) {
    const int x = i * kCellStride + j;
    const int64_t o = (int64_t)i * Mfull + j;
    const uint32_t ax = aux[o];
    const double v = cell_score_t(A.md, A.T, S.src_len[i], S.src_uniq[i], S.src_chars[i], S.tgt_len[j],
                                  S.tgt_uniq[j], S.tgt_chars[j], (int)(ax & 0xffu), out[o], S.covt[x],
                                  (int)(ax >> 8), kExpTableDev);
    if (kFeatures) {  // features_from_profiles (classifier.py:69-97), IEEE divisions
      const int cov = (int)(ax & 0xffu), sh = (int)(ax >> 8), covt = S.covt[x];
      const int Ls = S.src_len[i], Lt = S.tgt_len[j], Us = S.src_uniq[i], Ut = S.tgt_uniq[j];
      double *f = A.features + 6 * (A.b.pair_sim_off[p] + (int64_t)(i0 + i) * Mfull + (j0 + j));
      f[0] = clip4(fdiv((double)Ls, (double)Lt));
      f[1] = fdiv((double)cov, (double)Ls);
      f[2] = fdiv((double)covt, (double)Lt);
      f[3] = cov ? fdiv(out[o], (double)cov) : 0.0;
      f[4] = clip4(fdiv((double)S.src_chars[i], (double)S.tgt_chars[j]));
      f[5] = fdiv((double)sh, (double)(Us > Ut ? Us : Ut));
    }
    out[o] = v;
    if (fuse_nw) tile[i * 64 + j] = v;
    i += di;
    j += dj;
    if (j >= M) {
      j -= M;
      ++i;
    }
  }
  if (!fuse_nw) return;
  __syncthreads();
  // ---- NW fill + traceback + threshold filter on the tile (align.py:170-181,
  //      132-163, 323-332), one warp; the other warps are done
  if (warp == 0) {
    double *rowbuf = (double *)(smem_raw + kNwTileBytes);
    uint32_t *dirs = (uint32_t *)(smem_raw + kNwTileBytes + kNwRowBytes);
    nw_solve<kNwMine, false>(tile, 64, N, M, A.gap, A.mismatch, A.bonus, A.threshold, nullptr, dirs, rowbuf,
                             A.nw_matches + A.nw_out_off[p], nullptr, A.nw_counts + p,
                             A.nw_score ? A.nw_score + p : nullptr);
  }
}

}  // namespace bimine
