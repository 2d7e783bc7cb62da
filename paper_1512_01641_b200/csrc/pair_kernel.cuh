// pair_kernel.cuh -- score matrix of one document pair per CTA.
//
// build_score_matrix (align.py:102-129) for pairs with N, M <= 64 and
// sentences of <= 255 tokens (all C2/C4/C5 pairs); larger pairs (C1, C3)
// run the same kernel over 64x64 sentence tiles, (pair, i0, j0) per CTA.
// 8 warps, 4 CTAs per SM.
//
//  A  target side, warp per target sentence, lanes over its tokens: each
//     token goes into a shared open-addressing hash whose 64-bit slots
//     hold (token, dense id); the id is drawn from a counter by the thread
//     that claims the empty slot, so there is no separate numbering pass.
//     colmask[d] = 64-bit set of the chunk's target sentences holding
//     token d; a Bloom filter in front of the hash rejects most of the
//     dictionary translations that are absent.
//  D  warp per source sentence i (claimed longest first); lane j owns
//     target sentences j and j + 32.  The sentence's occurrences are cut
//     into segments of <= 32 occurrences whose dictionary rows (p > 0
//     entries, one 16-byte {p, t} record each) total <= 96 entries.  The
//     warp walks a segment's entries flattened, 32 per step, each lane
//     finding its occurrence by a 5-step shuffle search, so lanes stay busy
//     whatever the row lengths.  Each hit (entry target in the chunk) is
//     appended, in entry order, to the warp's candidate list as (colmask,
//     p), p negated on the first candidate of each occurrence, and sets
//     reachcol[d] |= bit i (reachable_targets, classifier.py:54-59).  A
//     candidate-major pass then keeps, per lane j, the best p of the
//     current occurrence; at each negated p the previous best is added to
//     the running sum and counted in `covered` when > 0 -- the exact
//     sequential sum of classifier.py:75-82 (an occurrence whose best is 0
//     would add +0.0 to a non-negative sum: skipping it is bit-identical).
//     Shared tokens (classifier.py:94): the first occurrence of each
//     distinct chunk token of the sentence (a per-warp seen bitmap over
//     dense ids) adds its colmask bits.
//  C  warp per target sentence j, lanes = occurrences (dense ids looked up
//     again): transposing the reachcol rows gives covered_target(i, j) by popc
//     (classifier.py:88-92), multiplicities included.
//  F  all threads, one cell each: six features -> margin -> logistic
//     (terms.cuh), one coalesced store per cell.  The running sums of D are
//     parked in the cell's own output slot (L2) and overwritten here.
//
// If the chunk's target side exceeds the hash capacity (1024 distinct
// tokens; chunks start at <= 2048 occurrences) it is processed in parts
// (same results, more passes).
#pragma once

#include "common.cuh"
#include "terms.cuh"

namespace bimine {

constexpr int kPairThreads = 256;
constexpr int kPairWarps = kPairThreads / 32;
constexpr int kPairMax = 64;         // sentences per side
constexpr int kPairMaxLen = 255;     // tokens per sentence (u8 counts)
constexpr int kCellStride = 64;      // per-cell arrays are [64][64]
constexpr int kPkHashBits = 11;      // 2048 hash slots
constexpr int kPkSlots = 1 << kPkHashBits;
constexpr int kPkCapU = 1024;        // distinct target tokens per chunk
constexpr int kPkCapT = 2048;        // target occurrences per chunk
constexpr int kBloomBits = 14;       // 16384-bit prefilter in front of the hash
constexpr unsigned long long kPkEmpty = ~0ull;

struct PairArgs {
  BatchDev b;
  DictDev d;
  Model md;
  TermTables T;
  double *sim;
  uint16_t *aux;            // per-cell scratch, same layout as sim: covered | shared << 8
  const int64_t *tiles;     // (pair, i0, j0) per tile of the pairs larger than 64x64
  int64_t n_tiles;          // CTAs [0, n_tiles) are tiles, the rest one pair each
  // features mode (extract_features, classifier.py:62-112): the six
  // features of every cell at features[6 * (pair_sim_off + i * M + j) + k]
  double *features;
  unsigned long long *next_item;  // the persistent CTAs' work counter (zeroed before the launch)
  // upload gate (bimine_mine_host; null: the data are in place): a counter
  // that grows as upload pieces land.  bimine_mine_host launches before the
  // host has looked at the batch, so each CTA derives the value it needs:
  // once the pair and sentence arrays are in (ready >= 1) it bounds-checks
  // its pair against these sizes -- skipping it if out of range, the host
  // reports the error -- and waits for the piece of its last token; token
  // piece k covers [piece_start[k], piece_start[k + 1]), k < n_pieces
  const int32_t *ready;
  int64_t n_sentences, n_tokens;
  int32_t n_pieces;
  const int64_t *piece_start;
};

__device__ __forceinline__ void wait_ready(const int32_t *ready, int want) {
  while (true) {
    int r;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(r) : "l"(ready) : "memory");
    if (r >= want) break;
    __nanosleep(256);
  }
}

constexpr int kSegItems = 96;   // dictionary entries examined per warp segment

struct PairSmem {
  unsigned long long hkey[kPkSlots];  // token << 32 | dense id; kPkEmpty
  uint64_t colmask[kPkCapU];
  uint64_t reachcol[kPkCapU];
  uint32_t bloom[(1 << kBloomBits) / 32];
  uint64_t c_m[kPairWarps][kSegItems];  // per warp: a segment's in-chunk translations: colmask
  double c_p[kPairWarps][kSegItems];    //   probability (negated: first of its occurrence)
  uint32_t seen[kPairWarps][kPkCapU / 32];  // dense ids met in the warp's source sentence
  int64_t src_off[64], tgt_off[64];
  int32_t src_len[64], src_uniq[64], src_chars[64];
  int32_t tgt_len[64], tgt_uniq[64], tgt_chars[64];
  unsigned long long te_max;          // self-gated launch: the block's largest token end
  int32_t misc[8];                    // 0 dense-id counter, 1 chunk end, 2 D claims, 3 C claims
  uint8_t src_order[64];              // source sentences, longest first (phase D claim order)
  uint8_t covt[64 * 64];
};

constexpr size_t kPairSmemBytes = sizeof(PairSmem);

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

__device__ __forceinline__ bool bloom_has(const uint32_t *bloom, int32_t key) {
  const uint32_t b = bloom_bit(key);
  return (bloom[b >> 5] >> (b & 31)) & 1u;
}

// The chunk's target hash: 512 buckets of four 64-bit slots (token << 32 |
// dense id; empty = all ones).  A slot is only ever claimed as the first
// empty slot of its bucket, so the filled slots of a bucket are a prefix:
// a lookup reads its bucket with two 16-byte loads and takes the first
// slot whose token matches -- either the key's slot, or (key -1 only) the
// first empty slot, whose id field reads -1 = absent.  A full bucket
// without the key continues in the next one (rare at <= 1024 keys).
constexpr int kPkBucketBits = kPkHashBits - 2;

__device__ __forceinline__ int pk_find(const unsigned long long *hkey, int32_t key) {
  uint32_t b = hash_slot(key, 32 - kPkBucketBits);
  while (true) {
    const ulonglong2 x = *reinterpret_cast<const ulonglong2 *>(hkey + 4 * b);
    const ulonglong2 y = *reinterpret_cast<const ulonglong2 *>(hkey + 4 * b + 2);
    int d = -2;
    if ((int32_t)(y.y >> 32) == key) d = (int)(uint32_t)y.y;
    if ((int32_t)(y.x >> 32) == key) d = (int)(uint32_t)y.x;
    if ((int32_t)(x.y >> 32) == key) d = (int)(uint32_t)x.y;
    if ((int32_t)(x.x >> 32) == key) d = (int)(uint32_t)x.x;
    if (d != -2) return d;
    if (y.y == kPkEmpty) return -1;
    b = (b + 1u) & ((1u << kPkBucketBits) - 1u);
  }
}

// lookup behind the Bloom prefilter (most dictionary translations are absent)
__device__ __forceinline__ int pk_find_f(const uint32_t *bloom, const unsigned long long *hkey, int32_t key) {
  return bloom_has(bloom, key) ? pk_find(hkey, key) : -1;
}

// insert `key` (if absent) and return its dense id.  The thread that finds
// the bucket's first empty slot draws the id and publishes key and id in
// one 64-bit CAS, so a reader never sees a key without its id; an id drawn
// by a thread that loses the CAS to the same key is never used (a hole).
__device__ __forceinline__ int pk_insert(unsigned long long *hkey, int *counter, int32_t key) {
  uint32_t b = hash_slot(key, 32 - kPkBucketBits);
  int d = -1;  // drawn once, kept across attempts
  while (true) {
    unsigned long long *bk = hkey + 4 * b;
    int k = 0;
    for (; k < 4; ++k) {
      unsigned long long cur = bk[k];
      if (cur == kPkEmpty) {
        if (d < 0) d = atomicAdd(counter, 1);
        const unsigned long long want = ((unsigned long long)(uint32_t)key << 32) | (uint32_t)d;
        cur = atomicCAS(&bk[k], kPkEmpty, want);
        if (cur == kPkEmpty) return d;
      }
      if ((int32_t)(cur >> 32) == key) return (int)(uint32_t)cur;
    }
    b = (b + 1u) & ((1u << kPkBucketBits) - 1u);
  }
}

// (bit != 0 && p > best) ? p : best, as one predicate: the bit test feeds
// the compare's predicate input
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

// One work item of the score kernel: items [0, n_tiles) are the 64x64
// tiles of large pairs (first, so the long pairs start early), the rest one
// pair each (pairs larger than 64x64 are skipped there: their tiles cover
// them).  Every exit is CTA-uniform.
// kFeatures: also write the six features per cell (bimine_features_batch);
// kPacked: the batch's token ids are in the 24-bit form
template <bool kFeatures, bool kPacked>
__device__ __forceinline__ void pair_item(const PairArgs &A, PairSmem &S, const int64_t item) {
  int64_t p;
  int i0 = 0, j0 = 0;
  const bool is_tile = item < A.n_tiles;
  if (is_tile) {
    p = A.tiles[3 * item];
    i0 = (int)A.tiles[3 * item + 1];
    j0 = (int)A.tiles[3 * item + 2];
  } else {
    p = item - A.n_tiles;
  }
  const bool self_gate = A.ready != nullptr;
  if (self_gate) {  // the pair and sentence arrays first
    if (threadIdx.x == 0) wait_ready(A.ready, 1);
    __syncthreads();
  }
  const int Nfull = A.b.pair_n[p], Mfull = A.b.pair_m[p];
  if (self_gate) {  // the pair's sentence ranges, before any of them is read
    const int64_t ps = A.b.pair_src[p], pt = A.b.pair_tgt[p];
    if (Nfull < 1 || Mfull < 1 || ps < 0 || pt < 0 || ps + Nfull > A.n_sentences || pt + Mfull > A.n_sentences)
      return;
  }
  if (!is_tile && (Nfull > kPairMax || Mfull > kPairMax)) return;
  // this CTA's block: source sentences [i0, i0 + N), target sentences [j0, j0 + M)
  const int N = min(kPairMax, Nfull - i0), M = min(kPairMax, Mfull - j0);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t s_first = A.b.pair_src[p] + i0, t_first = A.b.pair_tgt[p] + j0;
  const TokenViewT<kPacked> tokens{A.b.tokens.t32};
  const uint64_t *__restrict__ rowdesc = A.d.rowdesc;
  const DictEntry *__restrict__ dent = A.d.ent;
  const int64_t n_rows = A.d.n_rows;
  // the block's cell (i, j) lives at out[i * Mfull + j]; also the running-sum scratch
  double *__restrict__ out = A.sim + A.b.pair_sim_off[p] + (int64_t)i0 * Mfull + j0;
  uint16_t *__restrict__ aux = A.aux + A.b.pair_sim_off[p] + (int64_t)i0 * Mfull + j0;

  // ---- 0: sentence metadata
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
  if (self_gate) {  // every sentence non-empty and inside the tokens; the piece of the last token
    int64_t te = 0;
    bool bad = false;
    if (tid < N || (tid >= 64 && tid - 64 < M)) {
      const int64_t o = tid < N ? S.src_off[tid] : S.tgt_off[tid - 64];
      const int l = tid < N ? S.src_len[tid] : S.tgt_len[tid - 64];
      bad = l < 1 || o < 0 || o + l > A.n_tokens;
      te = o + l;
    }
    if (__syncthreads_or(bad)) return;
    // the block's largest end: warp maxima, then one shared maximum
    for (int o = 16; o > 0; o >>= 1) te = max(te, (int64_t)__shfl_xor_sync(kFull, (long long)te, o));
    if (tid == 0) S.te_max = 0ull;
    __syncthreads();
    if (lane == 0) atomicMax(&S.te_max, (unsigned long long)te);
    __syncthreads();
    if (tid == 0) {
      const int64_t x = (int64_t)S.te_max - 1;
      int j = 0;  // the piece holding token x
      while (j + 1 < A.n_pieces && A.piece_start[j + 1] <= x) ++j;
      wait_ready(A.ready, j + 2);
    }
    __syncthreads();
  }
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
    // ---- chunk [jc0, jc1): at most kPkCapT target occurrences
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
        const unsigned ok = __ballot_sync(kFull, j < M && run + x <= kPkCapT);
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
      if (tid == 0) {
        S.misc[0] = 0;
        S.misc[2] = 0;
        S.misc[3] = 0;
      }
      {  // clear the hash, the masks and the prefilter (16-byte stores)
        uint4 z = make_uint4(0u, 0u, 0u, 0u);
        uint4 e = make_uint4(~0u, ~0u, ~0u, ~0u);
        uint4 *hk = reinterpret_cast<uint4 *>(S.hkey);
        for (int k = tid; k < kPkSlots / 2; k += kPairThreads) hk[k] = e;
        uint4 *cm = reinterpret_cast<uint4 *>(S.colmask);
        for (int k = tid; k < kPkCapU / 2; k += kPairThreads) cm[k] = z;
        uint4 *rc = reinterpret_cast<uint4 *>(S.reachcol);
        for (int k = tid; k < kPkCapU / 2; k += kPairThreads) rc[k] = z;
        uint4 *bl = reinterpret_cast<uint4 *>(S.bloom);
        for (int k = tid; k < (1 << kBloomBits) / 128; k += kPairThreads) bl[k] = z;
      }
      __syncthreads();
      // ---- A: insert the chunk's target tokens: dense id, colmask bit, prefilter bit
      for (int jj = warp; jj < nj; jj += kPairWarps) {
        const int64_t off = S.tgt_off[jc0 + jj];
        const int L = S.tgt_len[jc0 + jj];
        uint32_t *cw = reinterpret_cast<uint32_t *>(S.colmask) + (jj >> 5);
        const uint32_t jbit = 1u << (jj & 31);
        for (int k = lane; k < L; k += 32) {
          const int32_t t = tokens[off + k];
          const int d = pk_insert(S.hkey, &S.misc[0], t);
          if (d < kPkCapU) atomicOr(cw + 2 * d, jbit);
          const uint32_t b = bloom_bit(t);
          atomicOr(&S.bloom[b >> 5], 1u << (b & 31));
        }
      }
      __syncthreads();
      if (S.misc[0] <= kPkCapU || nj == 1) break;
      jc1 = jc0 + nj / 2;  // too many distinct tokens: halve the chunk
      __syncthreads();
    }
    const int nj = jc1 - jc0;
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
      uint64_t *cm = &S.c_m[0][0] + cbase;
      uint32_t *seen = S.seen[warp];
      double *cp = &S.c_p[0][0] + cbase;
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
        const uint64_t rd = rowdesc[s_w];
        e0_w = (int64_t)(rd >> 24);
        rl_w = (int)(rd & 0xFFFFFFull);
      }
      while (i < N) {
        const int L = S.src_len[i];
        const unsigned long long ibit = 1ull << i;
        int cov_lo = 0, cov_hi = 0, sh_lo = 0, sh_hi = 0;
        double sum_lo = 0.0, sum_hi = 0.0;
        seen[lane] = 0u;  // (kPkCapU = 1024 dense ids: 32 words)
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
                const DictEntry en = dent[oeb + it];
                w_tgt[st] = en.t;
                w_p[st] = en.p;
              }
            }
          }
          // next window: the rest of this sentence, else the next sentence
          const bool more = seg + cnt < L;
          const int32_t tok_nx = more ? load_tok(i, seg + cnt) : load_tok(i_nxt, 0);
          // shared tokens: first occurrence of a source token that is a chunk
          // token (one lane of each distinct dense id claims its seen bit)
          const int ds = in_seg ? pk_find_f(S.bloom, S.hkey, s) : -1;
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
              double pr = 0.0;
              if (it < rl0) {
                const DictEntry en = dent[r0 + it];
                d = pk_find_f(S.bloom, S.hkey, en.t);
                pr = en.p;
              }
              const uint64_t m = d >= 0 ? S.colmask[d] : 0ull;
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
              const uint64_t rd = rowdesc[s_w];
              e0_w = (int64_t)(rd >> 24);
              rl_w = (int)(rd & 0xFFFFFFull);
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
                const DictEntry en = dent[oeb + it];
                tg = en.t;
                pr = en.p;
              }
            }
            const int d = tg >= 0 ? pk_find_f(S.bloom, S.hkey, tg) : -1;
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
            const uint64_t rd = rowdesc[s_w];
            e0_w = (int64_t)(rd >> 24);
            rl_w = (int)(rd & 0xFFFFFFull);
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
            const uint64_t rd = rowdesc[s_w];
            e0_w = (int64_t)(rd >> 24);
            rl_w = (int)(rd & 0xFFFFFFull);
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
      const int64_t off = S.tgt_off[jc0 + jj];
      const int L = S.tgt_len[jc0 + jj];
      int c_lo = 0, c_hi = 0;
      for (int seg = 0; seg < L; seg += 32) {
        // the occurrence's dense id again (every chunk token is in the hash)
        const uint64_t r = (seg + lane < L) ? S.reachcol[pk_find(S.hkey, tokens[off + seg + lane])] : 0ull;
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
  const int cells = N * M;
  // every integer-ratio term of the block in the tables? (the usual case:
  // no per-cell range tests)
  bool in_tables;
  {
    bool ok = true;
    if (tid < N) ok = S.src_len[tid] < kTermDim && S.src_uniq[tid] < kTermDim && S.src_chars[tid] < kCharDim;
    else if (tid >= 64 && tid - 64 < M)
      ok = S.tgt_len[tid - 64] < kTermDim && S.tgt_uniq[tid - 64] < kTermDim && S.tgt_chars[tid - 64] < kCharDim;
    in_tables = __syncthreads_and(ok);
  }
  // cell c = i * M + j, stepped without integer division
  const int di = kPairThreads / M, dj = kPairThreads - di * M;
  int i = tid / M, j = tid - (tid / M) * M;
  for (int c = tid; c < cells; c += kPairThreads) {
    const int x = i * kCellStride + j;
    const int64_t o = (int64_t)i * Mfull + j;
    const uint32_t ax = aux[o];
    const double v =
        in_tables ? cell_score_t<true>(A.md, A.T, S.src_len[i], S.src_uniq[i], S.src_chars[i], S.tgt_len[j],
                                       S.tgt_uniq[j], S.tgt_chars[j], (int)(ax & 0xffu), out[o], S.covt[x],
                                       (int)(ax >> 8), kExpTableDev)
                  : cell_score_t<false>(A.md, A.T, S.src_len[i], S.src_uniq[i], S.src_chars[i], S.tgt_len[j],
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
    i += di;
    j += dj;
    if (j >= M) {
      j -= M;
      ++i;
    }
  }
}

// Persistent CTAs (as many as are resident at once) take the items in order
// from a counter, so a CTA that finishes moves straight to the next item
// whose data has landed (bimine_mine_host's gated uploads), with no wave of
// newly dispatched CTAs waiting behind a piece still in flight.
template <bool kFeatures, bool kPacked>
__global__ void __launch_bounds__(kPairThreads, 4) pair_kernel(const PairArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PairSmem &S = *reinterpret_cast<PairSmem *>(smem_raw);
  __shared__ int64_t s_item;
  const int64_t n_items = A.n_tiles + A.b.n_pairs;
  while (true) {
    if (threadIdx.x == 0) s_item = (int64_t)atomicAdd(A.next_item, 1ull);
    __syncthreads();
    const int64_t item = s_item;
    if (item >= n_items) break;
    pair_item<kFeatures, kPacked>(A, S, item);
    __syncthreads();  // the item's shared-memory state is dead before the next one starts
  }
}

}  // namespace bimine
