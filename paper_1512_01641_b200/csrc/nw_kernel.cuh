// nw_kernel.cuh -- Needleman-Wunsch fill + traceback + threshold filter.
//
// Reference: nw_align / nw_align_wavefront (align.py:170-200) fill the
// table of the *reversed* score matrix (align.py:166-167) with
//   dp[a][b] = max(dp[a-1][b-1] + c, dp[a-1][b] - gap, dp[a][b-1] - gap)
//   c = mismatch + R[a-1][b-1] * (bonus - mismatch)
// where a strict `>` keeps the earlier candidate on ties
// (_nwcore.pyx:28-34), then walk forward from (0, 0) preferring the
// diagonal, then a source gap, then a target gap (align.py:132-163),
// and finally keep Match steps whose similarity reaches the threshold
// (align.py:323-332).
//
// Because the traceback's equality tests re-evaluate exactly the
// candidates the fill compared, "first candidate equal to the max in
// the order diag, up, left" is the candidate the fill kept; recording it
// as a 2-bit direction during the fill reproduces the reference walk
// without the float64 table (verified against the reference on the
// instance families of tests/golden/nw_golden.npz).
//
// One warp aligns one problem.  Rows of the reversed table are processed
// in bands of 32, lane l owning row a0 + 1 + l; at step s lane l computes
// column b = s - l + 1, so the 32 lanes sweep one anti-diagonal per step:
// "up" arrives from lane l-1 by a warp shuffle, "diagonal" is the value
// that arrived one step earlier, "left" is the lane's own previous cell.
// Row a0 (the band's upper boundary) comes from a per-warp row buffer
// that the previous band's lane 31 filled.  Directions (2 bits per cell,
// 16 cells per word) live in shared memory for problems that fit and in
// a per-warp global scratch slot otherwise; the walk runs on lane 0.
#pragma once

#include "common.cuh"

namespace bimine {

enum NwMode { kNwMine = 0, kNwSteps = 1, kNwTable = 2 };

struct NwArgs {
  const double *sim;           // all pairs, row-major per pair at sim_off
  const int64_t *sim_off;      // [pairs]
  const int32_t *pair_n;       // [pairs]
  const int32_t *pair_m;       // [pairs]
  const int64_t *problem_ids;  // [n_problems] or null (identity)
  int64_t n_problems;
  int32_t n_settings;          // problem q -> pair q / n_settings, setting q % n_settings
  const double *gap;           // [n_settings], or [n_problems] if gap_per_problem; null: gap1
  int gap_per_problem;
  const double *threshold;     // [n_settings] (mine mode); null: threshold1
  double gap1, threshold1;     // one setting passed by value
  int small_only;              // nw_kernel: skip pairs larger than 64 x 64 (a cluster launch takes them)
  double mismatch, bonus;
  // mine mode
  const int64_t *out_off;      // [problems] slot offsets
  bimine_match *matches;
  int32_t *counts;
  double *score;               // [problems] or null
  // steps mode
  const int64_t *step_off;
  uint8_t *steps;
  int32_t *n_steps;
  // table mode (single problem, reversed sim, caller boundaries)
  double *table;
  // scratch
  int dir_words_per_warp;      // capacity (u32 words) of each warp's direction area
  int row_doubles_per_warp;    // capacity of each warp's row buffer
  uint32_t *g_dirs;            // global scratch (null -> shared memory)
  double *g_rows;
};

__device__ __forceinline__ double nw_gap(const NwArgs &A, int64_t q, int setting) {
  return A.gap ? (A.gap_per_problem ? A.gap[q] : A.gap[setting]) : A.gap1;
}
__device__ __forceinline__ double nw_threshold(const NwArgs &A, int setting) {
  return A.threshold ? A.threshold[setting] : A.threshold1;
}

// One problem on one warp.  `sim` is the problem's row-major matrix with
// row stride `ld` (global memory, or a shared-memory tile in the fused
// score kernel); table mode reads the already reversed matrix.  Outputs:
// mine mode -> out[0..count) matches (i ascending), steps mode -> codes.
template <int MODE, bool kGlobal>
__device__ __forceinline__ void nw_solve(const double *__restrict__ sim, int ld, int N, int M, double gap,
                                         double mismatch, double bonus, double threshold, double *table,
                                         uint32_t *dirs, double *rowbuf, bimine_match *out, uint8_t *steps,
                                         int32_t *count_out, double *score_out) {
  const int lane = threadIdx.x & 31;
  const double ng = -gap;
  const double span = fsub(bonus, mismatch);
  const int stride = (M >> 4) + 1;  // direction words per row (cells b = 0..M)
  const int64_t tw = (int64_t)M + 1;

  // row 0 of the reversed table (kernels.py:46, or the caller's in table mode)
  for (int b = lane; b <= M; b += 32) rowbuf[b] = (MODE == kNwTable) ? table[b] : fmul(ng, (double)b);
  __syncwarp();
  double last = 0.0;  // dp[N][M], on the lane that owns row N
  for (int a0 = 0; a0 < N; a0 += 32) {
    const int a = a0 + 1 + lane;
    const bool active = a <= N;
    // dp[a][0] (kernels.py:47) and dp[a-1][0]
    const double left0 = (MODE == kNwTable) ? (active ? table[(int64_t)a * tw] : 0.0) : fmul(ng, (double)a);
    double cur = left0;
    double diag = 0.0;
    if (lane == 0) diag = rowbuf[0];
    {
      const double prev_row0 = __shfl_up_sync(kFull, left0, 1);
      if (lane > 0) diag = prev_row0;
    }
    // this lane's row of R: the reversed matrix row a-1 is sim row N - a
    // walked backwards (table mode receives the reversed matrix itself,
    // as kernels.fill_sequential passes it, kernels.py:55-57)
    const double *srow = (MODE == kNwTable) ? sim + (int64_t)(a - 1) * ld : sim + (int64_t)(N - a) * ld + (M - 1);
    const int64_t sdir = (MODE == kNwTable) ? 1 : -1;
    auto ldr = [&](int b) -> double {
      if (!(active && b >= 1 && b <= M)) return 0.0;
      const double *q = srow + sdir * (b - 1);
      return kGlobal ? __ldg(q) : *q;
    };
    uint32_t bits = 0u;
    const int nsteps = M + 31;
    // R values for 8 steps at a time, the next 8 prefetched into registers
    // (one dependent load per step would make the sweep latency bound)
    double cur8[8], nxt8[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) nxt8[u] = ldr(u - lane + 1);
    for (int s0 = 0; s0 < nsteps; s0 += 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) cur8[u] = nxt8[u];
#pragma unroll
      for (int u = 0; u < 8; ++u) nxt8[u] = ldr(s0 + 8 + u - lane + 1);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int s = s0 + u;
        if (s >= nsteps) break;
        const int b = s - lane + 1;
        double up = __shfl_up_sync(kFull, cur, 1);
        if (lane == 0) {
          up = (b >= 1 && b <= M) ? rowbuf[b] : 0.0;
          if (b >= 1 && b <= M) diag = rowbuf[b - 1];
        }
        if (active && b >= 1 && b <= M) {
          const double c = fadd(mismatch, fmul(cur8[u], span));
          double best = fadd(diag, c);
          uint32_t dir = 0u;
          double cand = fsub(up, gap);
          if (cand > best) {
            best = cand;
            dir = 1u;
          }
          cand = fsub(cur, gap);
          if (cand > best) {
            best = cand;
            dir = 2u;
          }
          cur = best;
          if (MODE == kNwTable) {
            table[(int64_t)a * tw + b] = best;
          } else {
            bits |= dir << (2 * (b & 15));
            if ((b & 15) == 15 || b == M) {
              dirs[(int64_t)a * stride + (b >> 4)] = bits;
              bits = 0u;
            }
          }
          if (lane == 31) rowbuf[b] = best;
          if (a == N && b == M) last = best;
        }
        if (lane > 0) diag = up;  // dp[a-1][b] becomes next step's diagonal
      }
    }
    // the next band's lane 0 needs dp[a0+32][0] as its first diagonal
    __syncwarp();
    if (lane == 31) rowbuf[0] = left0;
    __syncwarp();
  }
  // dp[N][M] lives on lane (N - 1) % 32
  last = __shfl_sync(kFull, last, (N - 1) & 31);
  if (MODE == kNwTable) return;
  if (lane == 0) {
    int a = N, b = M;
    int64_t cnt = 0;
    if (MODE == kNwMine) {
      while (a > 0 && b > 0) {
        const uint32_t d = (dirs[(int64_t)a * stride + (b >> 4)] >> (2 * (b & 15))) & 3u;
        if (d == 0u) {
          const int i = N - a, j = M - b;
          const double v = sim[(int64_t)i * ld + j];
          if (v >= threshold) {
            out[cnt].score = v;
            out[cnt].i = i;
            out[cnt].j = j;
            ++cnt;
          }
          --a;
          --b;
        } else if (d == 1u) {
          --a;
        } else {
          --b;
        }
      }
    } else {
      while (a > 0 && b > 0) {
        const uint32_t d = (dirs[(int64_t)a * stride + (b >> 4)] >> (2 * (b & 15))) & 3u;
        steps[cnt++] = (uint8_t)d;
        if (d == 0u) {
          --a;
          --b;
        } else if (d == 1u) {
          --a;
        } else {
          --b;
        }
      }
      while (a > 0) {
        steps[cnt++] = 1u;
        --a;
      }
      while (b > 0) {
        steps[cnt++] = 2u;
        --b;
      }
    }
    *count_out = (int32_t)cnt;
    if (score_out) *score_out = last;
  }
  __syncwarp();
}

// ---- the lean band sweep -------------------------------------------------
//
// One 32-row band (rows a0+1 .. a0+32 of the reversed table, lane l owns
// row a0+1+l) swept over all columns: at step s lane l computes column
// b = s - l + 1.  Everything that does not depend on the neighbour's
// value is prepared once per group of 8 steps, off the dependency chain:
// the 8 R values (loaded 8 steps ahead), c = mismatch + R * span, the
// valid-step mask and lane 0's 9 boundary values dp[a0][s0 .. s0+8]
// (from `top`, which may wait for a producer).  A step is then a shuffle,
// three adds, two compares and selects.  Directions: per lane and group
// one u16 (2 bits per step), dirs_band[group * 32 + lane] -- coalesced.
// The band's last row (lane 31) goes to `bot` one value per step.
// Returns the lane's final value dp[row][M] (cur after the sweep).
__host__ __device__ inline int nw_groups(int M) { return (M + 31 + 7) >> 3; }

// kDiag: `sim` is the band's block of the diagonal layout (nw_diag_kernel):
// entry [s][lane] = the lane's match/mismatch term c at step s, so a step
// reads 32 consecutive doubles (zeros outside the table)
template <bool kGlobal, class Top, class Bot, bool kDiag = false>
__device__ __forceinline__ double band_sweep(const double *__restrict__ sim, int ld, int N, int M, int a0, double gap,
                                             double mismatch, double span, Top &top, Bot &bot,
                                             uint16_t *__restrict__ dirs_band) {
  const int lane = threadIdx.x & 31;
  const int a = a0 + 1 + lane;
  const bool active = a <= N;
  const double ng = -gap;
  const double left0 = fmul(ng, (double)a);  // dp[a][0] (kernels.py:47)
  double cur = left0;
  double diag = __shfl_up_sync(kFull, left0, 1);  // dp[a-1][0] for lanes > 0
  const double *srow = sim + (int64_t)(N - (active ? a : N)) * ld + (M - 1);
  const int nsteps = M + 31;
  // the 8 values of the group starting at step t0: element u is column
  // b = t0 + u - lane + 1, at srow - (b - 1); one base pointer and one
  // validity mask per group, then predicated loads
  auto load_group = [&](int t0, double *dst) {
    const int bb = t0 - lane + 1;
    const uint32_t lim = active ? (uint32_t)M : 0u;  // column b valid iff (b - 1) < lim
    const double *q = srow - (bb - 1);
#pragma unroll
    for (int u = 0; u < 8; ++u)
      dst[u] = ((uint32_t)(bb + u - 1) < lim) ? (kGlobal ? __ldg(q - u) : *(q - u)) : 0.0;
  };
  double nxt[8];
  if (kDiag) {
#pragma unroll
    for (int u = 0; u < 8; ++u) nxt[u] = __ldg(sim + u * 32 + lane);
  } else {
    load_group(0, nxt);
  }
  for (int s0 = 0, grp = 0; s0 < nsteps; s0 += 8, ++grp) {
    double c[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) c[u] = kDiag ? nxt[u] : fadd(mismatch, fmul(nxt[u], span));
    if (kDiag) {
#pragma unroll
      for (int u = 0; u < 8; ++u) nxt[u] = __ldg(sim + (int64_t)(s0 + 8 + u) * 32 + lane);
    } else {
      load_group(s0 + 8, nxt);
    }
    // steps s0+u with 1 <= b <= M for this lane
    const int lo = max(lane - s0, 0), hi = min(lane + M - 1 - s0, 7);
    const uint32_t vmask = (active && lo <= hi) ? (((2u << hi) - 1u) & ~((1u << lo) - 1u)) : 0u;
    double rb[9];
    top.load9(s0, rb);  // lane 0: dp[a0][s0 .. s0+8]
    bot.reserve(s0);    // whole warp: room for this group's boundary values
    __syncwarp();       // reconverge before the shuffles of the step loop
    uint32_t bits = 0u;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      double up = __shfl_up_sync(kFull, cur, 1);
      if (lane == 0) {
        up = rb[u + 1];
        diag = rb[u];
      }
      double best = fadd(diag, c[u]);
      const double t1 = fsub(up, gap);
      const bool p1 = t1 > best;
      best = p1 ? t1 : best;
      const double t2 = fsub(cur, gap);
      const bool p2 = t2 > best;
      best = p2 ? t2 : best;
      const bool v = (vmask >> u) & 1u;
      cur = v ? best : cur;
      bits |= (p2 ? 2u : (p1 ? 1u : 0u)) << (2 * u);
      bot.put(s0 + u, v, best);  // lane 31's cell of row a0+32, column s0+u-30
      diag = up;
    }
    dirs_band[grp * 32 + lane] = (uint16_t)bits;
  }
  return cur;
}

// traceback direction of reversed cell (a, b) from band-sweep directions
__device__ __forceinline__ uint32_t lean_dir(const uint16_t *dirs, int G8, int a, int b) {
  const int g = (a - 1) >> 5, l = (a - 1) & 31, s = b + l - 1;
  return ((uint32_t)dirs[((int64_t)g * G8 + (s >> 3)) * 32 + l] >> (2 * (s & 7))) & 3u;
}

// boundary providers / consumers for band_sweep
struct TopAnalytic {  // row 0: -gap * b (kernels.py:46)
  double ng;
  __device__ void load9(int s0, double *rb) const {
#pragma unroll
    for (int u = 0; u < 9; ++u) rb[u] = fmul(ng, (double)(s0 + u));
  }
};
struct TopRow {  // a row buffer rowbuf[0..M] (the previous band's last row)
  const double *row;
  int M;
  __device__ void load9(int s0, double *rb) const {
#pragma unroll
    for (int u = 0; u < 9; ++u) rb[u] = row[min(s0 + u, M)];
  }
};
struct BotRow {  // lane 31 writes row[b] for the next band
  double *row;
  int M;
  bool on;
  __device__ void reserve(int) const {}
  __device__ void put(int s, bool v, double best) const {
    if (on && v && (threadIdx.x & 31) == 31) row[s - 30] = best;
  }
};
struct BotNone {
  __device__ void reserve(int) const {}
  __device__ void put(int, bool, double) const {}
};

// Single-warp solve of a problem that fits one warp's scratch: bands in
// sequence through a row buffer (M+1 doubles); directions in dirs
// (G * nw_groups(M) * 32 u16).
template <int MODE, bool kGlobal>
__device__ __forceinline__ void nw_solve_lean(const double *__restrict__ sim, int ld, int N, int M, double gap,
                                              double mismatch, double bonus, double threshold, uint16_t *dirs,
                                              double *rowbuf, bimine_match *out, uint8_t *steps, int32_t *count_out,
                                              double *score_out) {
  const int lane = threadIdx.x & 31;
  const double ng = -gap, span = fsub(bonus, mismatch);
  const int G = (N + 31) >> 5, G8 = nw_groups(M);
  double last = 0.0;
  for (int g = 0; g < G; ++g) {
    BotRow bot{rowbuf, M, g + 1 < G};
    double fin;
    if (g == 0) {
      TopAnalytic top{ng};
      fin = band_sweep<kGlobal>(sim, ld, N, M, 0, gap, mismatch, span, top, bot, dirs);
    } else {
      TopRow top{rowbuf, M};
      // the band reads rowbuf[b] before lane 31 of the same sweep could
      // overwrite it: reads of column s0+8 happen at group s0, writes of
      // column s0+u-30 later -- never the same column within a group
      fin = band_sweep<kGlobal>(sim, ld, N, M, 32 * g, gap, mismatch, span, top, bot, dirs + (int64_t)g * G8 * 32);
    }
    if (32 * g + 1 + lane == N) last = fin;
    __syncwarp();
    if (lane == 31 && g + 1 < G) rowbuf[0] = fmul(ng, (double)(32 * g + 32));  // dp[32g+32][0]
    __syncwarp();
  }
  last = __shfl_sync(kFull, last, (N - 1) & 31);
  // the walk (lane 0): branch-free position updates; mine mode only records
  // the Match cells -- their similarities are gathered by the whole warp
  // afterwards, so no global load sits on the walk's dependency chain
  int cnt = 0;
  if (lane == 0) {
    int a = N, b = M;
    while (a > 0 && b > 0) {
      const uint32_t d = lean_dir(dirs, G8, a, b);
      if (MODE == kNwMine) {
        if (d == 0u) {
          out[cnt].i = N - a;
          out[cnt].j = M - b;
          ++cnt;
        }
      } else {
        steps[cnt++] = (uint8_t)d;
      }
      a -= (d != 2u);
      b -= (d != 1u);
    }
    if (MODE != kNwMine) {
      while (a > 0) {
        steps[cnt++] = 1u;
        --a;
      }
      while (b > 0) {
        steps[cnt++] = 2u;
        --b;
      }
    }
  }
  cnt = __shfl_sync(kFull, cnt, 0);
  __syncwarp();
  if (MODE == kNwMine) {  // keep matches with sim >= threshold, in order (align.py:323-332)
    int kept = 0;
    for (int base = 0; base < cnt; base += 32) {
      const int c = base + lane;
      double v = 0.0;
      int32_t i = 0, j = 0;
      if (c < cnt) {
        i = out[c].i;
        j = out[c].j;
        v = sim[(int64_t)i * ld + j];
      }
      const bool keep = c < cnt && v >= threshold;
      const unsigned bal = __ballot_sync(kFull, keep);
      __syncwarp();
      if (keep) {
        bimine_match &o = out[kept + __popc(bal & ((1u << lane) - 1u))];
        o.score = v;
        o.i = i;
        o.j = j;
      }
      kept += __popc(bal);
      __syncwarp();
    }
    cnt = kept;
  }
  if (lane == 0) {
    *count_out = (int32_t)cnt;
    if (score_out) *score_out = last;
  }
  __syncwarp();
}

__host__ __device__ inline int64_t lean_dir_words16(int N, int M) {
  return (int64_t)((N + 31) >> 5) * nw_groups(M) * 32;
}

template <int MODE>
__device__ void nw_problem(const NwArgs &A, int64_t q, uint32_t *dirs, double *rowbuf) {
  const int64_t pair = q / A.n_settings;
  const int setting = (int)(q % A.n_settings);
  const int N = A.pair_n[pair], M = A.pair_m[pair];
  if (A.small_only && (N > 64 || M > 64)) return;  // the cluster launch's
  const double gap = nw_gap(A, q, setting);
  const double thr = (MODE == kNwMine) ? nw_threshold(A, setting) : 0.0;
  bimine_match *out = (MODE == kNwMine) ? A.matches + A.out_off[q] : nullptr;
  uint8_t *st = (MODE == kNwSteps) ? A.steps + A.step_off[q] : nullptr;
  int32_t *cnt = (MODE == kNwMine) ? A.counts + q : (MODE == kNwSteps) ? A.n_steps + q : nullptr;
  int32_t dummy;
  if (MODE == kNwTable)
    nw_solve<MODE, true>(A.sim + A.sim_off[pair], M, N, M, gap, A.mismatch, A.bonus, thr, A.table, dirs, rowbuf, out,
                         st, cnt ? cnt : &dummy, A.score ? A.score + q : nullptr);
  else
    nw_solve_lean<MODE, true>(A.sim + A.sim_off[pair], M, N, M, gap, A.mismatch, A.bonus, thr, (uint16_t *)dirs,
                              rowbuf, out, st, cnt ? cnt : &dummy, A.score ? A.score + q : nullptr);
}

// Warps loop over problems; each warp owns one direction area and one
// row buffer, in dynamic shared memory (g_dirs == null) or in a global
// scratch slot.
template <int MODE>
__global__ void __launch_bounds__(128, 5) nw_kernel(const NwArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5;
  const int warps_per_block = blockDim.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * warps_per_block + warp;
  const int64_t total_warps = (int64_t)gridDim.x * warps_per_block;
  uint32_t *dirs;
  double *rowbuf;
  if (A.g_dirs) {
    dirs = A.g_dirs + gw * A.dir_words_per_warp;
    rowbuf = A.g_rows + gw * A.row_doubles_per_warp;
  } else {
    double *rows = (double *)smem_raw;
    uint32_t *dr = (uint32_t *)(rows + (size_t)warps_per_block * A.row_doubles_per_warp);
    rowbuf = rows + (size_t)warp * A.row_doubles_per_warp;
    dirs = dr + (size_t)warp * A.dir_words_per_warp;
  }
  for (int64_t k = gw; k < A.n_problems; k += total_warps) {
    const int64_t q = A.problem_ids ? A.problem_ids[k] : k;
    nw_problem<MODE>(A, q, dirs, rowbuf);
  }
}

// ---- order-preserving compaction of per-problem match slots ----------

// Single CTA exclusive scan of counts -> base (int64) and total.
__global__ void __launch_bounds__(1024) scan_counts_kernel(const int32_t *counts, int64_t n, int64_t *base,
                                                           int64_t *total) {
  __shared__ int64_t part[1024];
  const int t = threadIdx.x;
  const int64_t per = (n + 1023) / 1024;
  const int64_t lo = min(n, t * per), hi = min(n, lo + per);
  int64_t s = 0;
  for (int64_t k = lo; k < hi; ++k) s += counts[k];
  part[t] = s;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const int64_t v = t >= o ? part[t - o] : 0;
    __syncthreads();
    part[t] += v;
    __syncthreads();
  }
  int64_t run = part[t] - s;
  for (int64_t k = lo; k < hi; ++k) {
    base[k] = run;
    run += counts[k];
  }
  if (t == 1023) *total = part[1023];
}

__global__ void gather_matches_kernel(const bimine_match *slots, const int64_t *out_off, const int32_t *counts,
                                      const int64_t *base, int64_t n, bimine_match *compact) {
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= n) return;
  const bimine_match *src = slots + out_off[w];
  bimine_match *dst = compact + base[w];
  for (int k = lane; k < counts[w]; k += 32) dst[k] = src[k];
}

}  // namespace bimine

namespace bimine {

// ---- tuning agreement (tuning.py:60-82) ------------------------------------
//
// alignment_agreement(candidate, reference): NW over the two index-pair
// lists with exact-equality scoring (match +1, mismatch -1, gap 1,
// _AGREEMENT_CONFIG tuning.py:28), counting Match steps that join equal
// pairs.  One warp per (pair, setting); the candidate list is the mining
// NW's match slots of that problem, the reference list the pair's
// human-aligned indices.  Same reversed fill / tie order / traceback as
// nw_problem (all values are small integers, exact in binary64).
struct AgreeArgs {
  const bimine_match *matches;
  const int64_t *out_off;
  const int32_t *counts;
  int64_t n_problems;
  int32_t n_settings;
  const int32_t *ref_ij;   // (i, j) int32 pairs
  const int64_t *ref_off;  // [pairs] first pair
  const int32_t *ref_len;  // [pairs]
  int32_t *matched;        // [problems]
  int64_t dir_words_per_warp;
  int64_t row_doubles_per_warp;
  double *g_rows;          // global scratch per launched warp (null: shared memory)
  uint32_t *g_dirs;
};

__device__ __forceinline__ bool agree_eq(const bimine_match *cand, const int32_t *ref, int a, int b) {
  return cand[a].i == ref[2 * b] && cand[a].j == ref[2 * b + 1];
}

__device__ void agree_problem(const AgreeArgs &A, int64_t q, double *rowbuf, uint32_t *dirs);

// Warps loop over (pair, setting) problems; each warp's row buffer and
// direction table sit in dynamic shared memory, or (lists too long for it)
// in a global scratch slot per launched warp.
__global__ void __launch_bounds__(128) agree_kernel(const AgreeArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  double *rowbuf;
  uint32_t *dirs;
  if (A.g_rows) {
    rowbuf = A.g_rows + gw * A.row_doubles_per_warp;
    dirs = A.g_dirs + gw * A.dir_words_per_warp;
  } else {
    rowbuf = (double *)smem_raw + (size_t)warp * A.row_doubles_per_warp;
    dirs = (uint32_t *)((double *)smem_raw + (size_t)(blockDim.x >> 5) * A.row_doubles_per_warp) +
           (size_t)warp * A.dir_words_per_warp;
  }
  for (int64_t q = gw; q < A.n_problems; q += nw) agree_problem(A, q, rowbuf, dirs);
}

__device__ void agree_problem(const AgreeArgs &A, int64_t q, double *rowbuf, uint32_t *dirs) {
  const int lane = threadIdx.x & 31;
  const int64_t pair = q / A.n_settings;
  const int K = A.counts[q];
  const int R = A.ref_len[pair];
  if (K == 0 || R == 0) {  // handled on the host (tuning.py:69-72)
    if (lane == 0) A.matched[q] = 0;
    return;
  }
  const bimine_match *cand = A.matches + A.out_off[q];
  const int32_t *ref = A.ref_ij + 2 * A.ref_off[pair];
  const double gap = 1.0, ng = -1.0;
  const int stride = (R >> 4) + 1;
  for (int b = lane; b <= R; b += 32) rowbuf[b] = fmul(ng, (double)b);
  __syncwarp();
  for (int a0 = 0; a0 < K; a0 += 32) {
    const int a = a0 + 1 + lane;
    const bool active = a <= K;
    const double left0 = fmul(ng, (double)a);
    double cur = left0;
    double diag = rowbuf[0];
    {
      const double prev_row0 = __shfl_up_sync(kFull, left0, 1);
      if (lane > 0) diag = prev_row0;
    }
    uint32_t bits = 0u;
    for (int s = 0; s < R + 31; ++s) {
      const int b = s - lane + 1;
      double up = __shfl_up_sync(kFull, cur, 1);
      if (lane == 0) {
        up = (b >= 1 && b <= R) ? rowbuf[b] : 0.0;
        if (b >= 1 && b <= R) diag = rowbuf[b - 1];
      }
      if (active && b >= 1 && b <= R) {
        // reversed problem: R[a-1][b-1] = sim[K-a][R-b]; c = -1 + sim * 2
        const double c = agree_eq(cand, ref, K - a, R - b) ? 1.0 : -1.0;
        double best = fadd(diag, c);
        uint32_t dir = 0u;
        double cand_v = fsub(up, gap);
        if (cand_v > best) {
          best = cand_v;
          dir = 1u;
        }
        cand_v = fsub(cur, gap);
        if (cand_v > best) {
          best = cand_v;
          dir = 2u;
        }
        cur = best;
        bits |= dir << (2 * (b & 15));
        if ((b & 15) == 15 || b == R) {
          dirs[(int64_t)a * stride + (b >> 4)] = bits;
          bits = 0u;
        }
        if (lane == 31) rowbuf[b] = best;
      }
      if (lane > 0) diag = up;
    }
    __syncwarp();
    if (lane == 31) rowbuf[0] = left0;
    __syncwarp();
  }
  if (lane == 0) {
    int a = K, b = R, m = 0;
    while (a > 0 && b > 0) {
      const uint32_t d = (dirs[(int64_t)a * stride + (b >> 4)] >> (2 * (b & 15))) & 3u;
      if (d == 0u) {
        if (agree_eq(cand, ref, K - a, R - b)) ++m;
        --a;
        --b;
      } else if (d == 1u) {
        --a;
      } else {
        --b;
      }
    }
    A.matched[q] = m;
  }
  __syncwarp();  // the warp's scratch is reused by its next problem
}

}  // namespace bimine

namespace bimine {

// ---- large problems: one CTA, warps pipelined over 32-row bands ----------
//
// For pairs too big for a warp's shared memory (C1 200x220, C3 4096x4096):
// band g (rows 32g+1 .. 32g+32 of the reversed table) runs on warp g % W
// with the same lane-per-row anti-diagonal sweep as nw_solve; the band's
// upper boundary (row 32g) streams from the warp that owns band g-1
// through a per-boundary shared-memory ring (producer/consumer positions,
// monotonic across the bands that reuse the ring), so W bands advance
// together a few columns apart.  Each lane prefetches its sim row into L1
// a line ahead (prefetch.global.L1) and loads it 8 steps ahead into
// registers.  Directions are stored per (band, step) as two ballot words
// (bit l = lane l's cell), written coalesced; the traceback walks them on
// lane 0 from a 64-step window staged by the whole warp, and the match
// scores are gathered in parallel afterwards.
#ifndef BIMINE_BIG_W
#define BIMINE_BIG_W 8
#endif
constexpr int kBigW = BIMINE_BIG_W;  // warps per CTA of the band pipeline (one per SM sub-partition)
#ifndef BIMINE_RING
#define BIMINE_RING 128
#endif
constexpr int kRing = BIMINE_RING;  // boundary values buffered per ring

// A ring slot carries its value and the position it holds, written by one
// 16-byte shared-memory store, so a consumer polling the slot's position
// sees a consistent value without any fence (a __threadfence_block per step
// would wait for the warp's outstanding global direction stores).
#ifndef BIMINE_SPIN_NS
#define BIMINE_SPIN_NS 0
#endif
constexpr unsigned kSpinNs = BIMINE_SPIN_NS;  // back-off of the band pipeline's spin waits (0: none;
                                              // measured: any back-off slows the pipeline)

struct BigRing {
  double2 slot[kRing];      // .x = value, .y = position bits (as double bits)
  volatile long long cons;  // positions consumed (capacity hint for the producer)
};

// The band pipeline's boundary store: lane 31's store of each step as one
// predicated generic instruction (no branch, so no reconvergence point in
// the step loop; every lane forms the address, only the predicate
// differs).  Generic addressing reaches the CTA's own ring, the next CTA's
// ring (a mapa'd address) and the global wrap row alike.
__device__ __forceinline__ void st_generic_v2_if(bool p, const void *slot, double v, long long tag) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %0, 0;\n\t@q st.relaxed.gpu.v2.f64 [%1], {%2, %3};\n\t}" ::"r"(
                   (unsigned)p),
               "l"(slot), "d"(v), "d"(__longlong_as_double(tag))
               : "memory");
}
// generic address of the same shared-memory object in cluster CTA `rank`
__device__ __forceinline__ void *cluster_generic(const void *p, unsigned rank) {
  void *r;
  asm volatile("mapa.u64 %0, %1, %2;" : "=l"(r) : "l"(p), "r"(rank));
  return r;
}
// %laneid, read once (a `threadIdx.x & 31` inside the step loop is
// re-derived from %tid by an S2R per use)
__device__ __forceinline__ unsigned lane_id_reg() {
  unsigned r;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(r));
  return r;
}

__device__ __forceinline__ double ring_get(const double2 *slot, long long pos) {
  double v, t;
  do {
    asm volatile("ld.volatile.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v), "=d"(t)
                 : "r"((unsigned)__cvta_generic_to_shared(slot))
                 : "memory");
  } while (__double_as_longlong(t) != pos);
  return v;
}

// Tagged-slot boundary provider (lane 0 of band g).  kShared: the slots
// are a shared-memory ring; the group's 9 slots are read together and those
// whose tag is not yet the wanted position re-read until the producer has
// written them; then `cons` releases what will not be read again.  Else a
// full global row (L2 round trips): the next group's slots are prefetched
// while the current group computes, and checked at the next group start.  Tags compare on their
// low 32 bits -- stale tags are at most a ring or two generations old.
template <bool kShared>
struct TopTagged {
  const double2 *buf;
  volatile long long *cons;  // ring only
  long long base;            // position of column 0 of this band's generation
  int M;
  double row0;               // dp[32g][0]
  double pv[9];
  int pt[9];
  __device__ __forceinline__ void ld(int b, double &v, int &t) const {
    double td;
    if (kShared) {
      const double2 *q = buf + ((base + b) & (kRing - 1));
      asm volatile("ld.volatile.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v), "=d"(td)
                   : "r"((unsigned)__cvta_generic_to_shared(q))
                   : "memory");
    } else {
      asm volatile("ld.relaxed.gpu.global.v2.f64 {%0, %1}, [%2];" : "=d"(v), "=d"(td) : "l"(buf + b) : "memory");
    }
    t = __double2loint(td);
  }
  __device__ __forceinline__ void fetch(int s0) {
#pragma unroll
    for (int u = 0; u < 9; ++u) {
      const int b = min(s0 + u, M);
      if (b == 0) {
        pv[u] = row0;
        pt[u] = (int)base;
      } else {
        ld(b, pv[u], pt[u]);
      }
    }
  }
  __device__ __forceinline__ void load9(int s0, double *rb) {
    if ((threadIdx.x & 31) != 0) return;
    if (kShared) {  // shared ring: ~30-cycle round trip, no prefetch state kept
#pragma unroll
      for (int u = 0; u < 9; ++u) {
        const int b = min(s0 + u, M);
        int t;
        if (b == 0) {
          rb[u] = row0;
          t = (int)base;
        } else {
          ld(b, rb[u], t);
        }
        pt[u] = t;
      }
#pragma unroll
      for (int u = 0; u < 9; ++u) {
        const int b = min(s0 + u, M);
        while (pt[u] != (int)(base + b)) {
          if (kSpinNs) __nanosleep(kSpinNs);
          ld(b, rb[u], pt[u]);
        }
      }
      *cons = base + min(s0 + 8, M);  // columns below s0+8 are not read again
      return;
    }
    if (s0 == 0) fetch(0);
#pragma unroll
    for (int u = 0; u < 9; ++u) {
      const int b = min(s0 + u, M);
      const int want = (int)(base + b);
      while (pt[u] != want) {
        if (kSpinNs) __nanosleep(kSpinNs);
        ld(b, pv[u], pt[u]);
      }
      rb[u] = pv[u];
    }
    fetch(s0 + 8);
  }
};

struct BotRing {
  BigRing *out;
  long long base;
  int M;
  bool on;
  bool l31;                       // this thread is lane 31
  long long seen = -(1ll << 62);  // last `cons` read (it only grows: a stale value is safe)
  // warp-uniform wait (every lane reads the same `cons`): the group's
  // stores, positions up to base + s0 + 7 - 30, must not lap the consumer;
  // `cons` is re-read only when the last value read does not allow them
  __device__ void reserve(int s0) {
    if (!on) return;
    const long long last = base + (s0 + 7 - 30);
    while (last - seen >= kRing - 1) {
      seen = out->cons;
      if (kSpinNs && last - seen >= kRing - 1) __nanosleep(kSpinNs);
    }
  }
};

// Boundaries between bands of the same round (warp w-1 -> warp w, w >= 1)
// stream through a shared-memory ring; the wrap-around boundary (warp W-1
// -> warp 0's next band) goes through a full row of tagged slots in global
// memory, double-buffered by generation parity: warp 0 starts that band only
// after finishing its previous one, so a bounded buffer there would tie band
// 0's progress to its own successors (a wait cycle once M exceeds the
// chain's total buffering).  With the wrap row never full, every wait points
// to a lower band or to a band of the same round further right -- acyclic.
struct BotRowG {  // lane 31 writes tagged slots of a global row
  double2 *row;
  long long base;
  bool on;
  bool l31;
  __device__ void reserve(int) const {}
};

template <int W>
constexpr size_t big_smem_bytes() { return W * sizeof(BigRing); }

// Diagonal layout of a problem's band g: steps s = 0 .. nw_diag_steps(M)-1
// (M + 31 rounded up to the group size, plus one prefetch group), 32 lanes.
__host__ __device__ inline int64_t nw_diag_steps(int M) { return (int64_t)((M + 31 + 7) & ~7) + 8; }

// One pass per large pair: c = mismatch + R[a-1][b-1] * (bonus - mismatch)
// (the sweep's two IEEE ops, kernels.py:47-52 / _nwcore.pyx:27) stored at
// [g][s][l] for reversed row a = 32g + 1 + l, column b = s - l + 1, so a
// warp step of the sweep reads 32 consecutive doubles.
__global__ void __launch_bounds__(256) nw_diag_kernel(const double *__restrict__ sim_all,
                                                       const int64_t *__restrict__ sim_off,
                                                       const int32_t *__restrict__ pair_n,
                                                       const int32_t *__restrict__ pair_m,
                                                       const int64_t *__restrict__ pairs,
                                                       const int64_t *__restrict__ diag_off, int64_t n_pairs,
                                                       double mismatch, double span, double *__restrict__ diag_all) {
  for (int64_t ps = blockIdx.z; ps < n_pairs; ps += gridDim.z) {  // distinct pairs
    const int64_t pair = pairs[ps];
    const int N = pair_n[pair], M = pair_m[pair];
    const double *__restrict__ sim = sim_all + sim_off[pair];
    const int64_t S = nw_diag_steps(M);
    for (int g = blockIdx.y; 32 * g < N; g += gridDim.y) {
      double *__restrict__ out = diag_all + diag_off[ps] + (int64_t)g * S * 32;
      for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < S * 32;
           x += (int64_t)gridDim.x * blockDim.x) {
        const int l = (int)(x & 31);
        const int64_t st = x >> 5;
        const int a = 32 * g + 1 + l;
        const int64_t b = st - l + 1;
        double v = 0.0;
        if (a <= N && b >= 1 && b <= M) v = fadd(mismatch, fmul(sim[(int64_t)(N - a) * M + (M - b)], span));
        out[x] = v;
      }
    }
  }
}

// Uniform per-problem scratch offsets (the layout of launch_nw's exact
// host offsets: [layouts] pair ids | layout offsets | per problem: layout,
// directions, wrap rows).  Listed problems get a layout each; without a
// list, problem q = pair * n_settings + setting shares its pair's.
__global__ void uniform_offsets_kernel(const int64_t *__restrict__ ids, int64_t n, int32_t n_settings, int64_t nd,
                                       int64_t dir_stride, int64_t rows_stride, int64_t diag_stride,
                                       int64_t *__restrict__ offs) {
  int64_t *pairs = offs, *pdoff = offs + nd, *doff = pdoff + nd, *dir = doff + n, *rows = dir + n;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t layout = ids ? k : k / n_settings;
    if (ids) {
      pairs[k] = ids[k] / n_settings;
      pdoff[k] = k * diag_stride;
    } else if (k % n_settings == 0) {
      pairs[layout] = layout;
      pdoff[layout] = layout * diag_stride;
    }
    doff[k] = layout * diag_stride;
    dir[k] = k * dir_stride;
    rows[k] = k * rows_stride;
  }
}

// Large problems: one thread-block cluster of K CTAs x W warps per problem.
// Band g runs on CTA (g / W) mod K, warp g mod W, round g / (W K).  The
// boundary into warp w of a CTA is that CTA's shared-memory ring w: rings
// 1..W-1 are written by the CTA's own warps, ring 0 by the last warp of the
// previous CTA of the cluster through distributed shared memory
// (st.shared::cluster; the producer polls the consumer's remote `cons`).
// The wrap-around boundary (last warp of CTA K-1 -> warp 0 of CTA 0, next
// round) is a full global row of tagged slots, double-buffered by round
// parity.  Every capacity wait points to a band of the same round further
// right and ends at the wrap row, which never waits, and every data wait to
// a lower band: the wait graph is acyclic for any N, M, K.  A cluster is
// co-scheduled, so all of a problem's CTAs are resident together.  After a
// cluster barrier, CTA 0 walks the traceback.
__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cluster_size() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same shared-memory object in CTA `rank`
__device__ __forceinline__ unsigned cluster_addr(const void *p, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"((unsigned)__cvta_generic_to_shared(p)), "r"(rank));
  return r;
}

struct BotRemote {  // lane 31 writes ring 0 of the next CTA of the cluster
  unsigned slot0;   // shared::cluster address of its slot[0]
  unsigned cons;    // shared::cluster address of its cons
  long long base;
  bool on;
  bool l31;
  long long seen = -(1ll << 62);  // last remote `cons` read (a DSMEM round trip per group otherwise)
  __device__ void reserve(int s0) {
    if (!on) return;
    const long long last = base + (s0 + 7 - 30);
    while (last - seen >= kRing - 1) {
      asm volatile("ld.relaxed.cluster.shared::cluster.b64 %0, [%1];" : "=l"(seen) : "r"(cons) : "memory");
      if (kSpinNs && last - seen >= kRing - 1) __nanosleep(kSpinNs);
    }
  }
};

#ifdef BIMINE_PROF_GLOBAL
__device__ unsigned long long g_prof_band[4096];
#endif
#ifdef BIMINE_FAKE_CALL
__device__ __noinline__ void bimine_noop_call(int g) { asm volatile("" ::"r"(g) : "memory"); }
#endif

template <int MODE, int W>
__global__ void __launch_bounds__(W * 32) nw_big_kernel(const NwArgs A, uint32_t *g_dirs_all,
                                                        const int64_t *dir_off, double2 *g_rows,
                                                        const int64_t *rows_off, double *last_val,
                                                        const double *diag_all, const int64_t *diag_off) {
  extern __shared__ __align__(16) unsigned char big_smem[];
  BigRing *rings = (BigRing *)big_smem;  // [W], ring w feeds warp w
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int crank = (int)cluster_rank(), K = (int)cluster_size();
  const int64_t slot = blockIdx.x / K;
  const int64_t q = A.problem_ids ? A.problem_ids[slot] : slot;
  const int64_t pair = q / A.n_settings;
  const int setting = (int)(q % A.n_settings);
  const int N = A.pair_n[pair], M = A.pair_m[pair];
  const double gap = nw_gap(A, q, setting);
  const double ng = -gap, mismatch = A.mismatch, span = fsub(A.bonus, A.mismatch);
  const int G = (N + 31) >> 5, G8 = nw_groups(M);
  uint16_t *dirs = (uint16_t *)(g_dirs_all + dir_off[slot]);  // [G][G8][32]
  double2 *wrap = g_rows + rows_off[slot];                    // [2][M+1] tagged, pre-filled with tag -1
  const long long W1 = (long long)M + 1;
  const int per_round = W * K;
  // [G][nw_diag_steps(M)][32]: the problem's pair's block of the operand layout
  const double *__restrict__ diag = diag_all + diag_off[slot];
  const int64_t dstride = nw_diag_steps(M) * 32;
#if defined(BIMINE_NW_PROFILE) || defined(BIMINE_PROF_ENTRY)
  if (threadIdx.x == 0) {
    unsigned long long gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    printf("prof entry cta %d ns %llu\n", crank, gt);
  }
#endif
  for (int k = threadIdx.x; k < W * kRing; k += blockDim.x)
    rings[k / kRing].slot[k % kRing] = make_double2(0.0, __longlong_as_double(-1ll));
  if (threadIdx.x < W) rings[threadIdx.x].cons = 0;
  __syncthreads();
  cluster_barrier();  // every ring initialised before any remote write
#ifdef BIMINE_PROF_GLOBAL
  if (crank == 0 && threadIdx.x == 0) {
    unsigned long long gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    g_prof_band[4095] = gt;
  }
#endif
#if defined(BIMINE_NW_PROFILE) || defined(BIMINE_PROF_START)
  if (threadIdx.x == 0) {
    unsigned long long gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    printf("prof start cta %d ns %llu\n", crank, gt);
  }
#endif
  const bool has_next = crank + 1 < K;
  const bool l31 = lane_id_reg() == 31u;
  const unsigned r_slot0 = has_next ? cluster_addr(&rings[0].slot[0], crank + 1) : 0u;
  const unsigned r_cons = has_next ? cluster_addr((const void *)&rings[0].cons, crank + 1) : 0u;
  void *const r_gslot0 = has_next ? cluster_generic(&rings[0].slot[0], crank + 1) : nullptr;
  for (int g = crank * W + warp, gen = 0; g < G; g += per_round, ++gen) {
    double fin;
    const bool last_warp = warp + 1 == W;
    const int ogr = (g + 1) / per_round;  // round of the consumer band
    BotRing bring{&rings[(warp + 1) % W], (long long)gen * W1, M, g + 1 < G && !last_warp, l31};
    BotRemote brem{r_slot0, r_cons, (long long)gen * W1, g + 1 < G && last_warp && has_next, l31};
    BotRowG brow{wrap + (ogr & 1) * W1, (long long)(g + 1) * W1, g + 1 < G && last_warp && !has_next, l31};
    // whichever of the three the band writes, one generic 16-byte store per
    // step: slot (b + off) & mask of `to`, tag base + b (b = s - 30)
    struct Bot3 {
      BotRing &r;
      BotRemote &x;
      char *to;
      int off, mask;
      long long base;
      bool on, l31;
      __device__ void reserve(int s0) {
        r.reserve(s0);
        x.reserve(s0);
      }
      __device__ void put(int s_, bool v, double best) const {
        const int b = s_ - 30;
        st_generic_v2_if(on && v && l31, to + (int64_t)((b + off) & mask) * 16, best, base + b);
      }
    };
    Bot3 bot{bring, brem, nullptr, 0, -1, 0, false, l31};
    if (bring.on) {
      bot.to = (char *)&bring.out->slot[0];
      bot.base = bring.base;
    } else if (brem.on) {
      bot.to = (char *)r_gslot0;
      bot.base = brem.base;
    } else if (brow.on) {
      bot.to = (char *)brow.row;
      bot.base = brow.base;
    }
    bot.on = bring.on || brem.on || brow.on;
    if (!brow.on) {  // a ring: slots wrap
      bot.off = (int)(bot.base & (kRing - 1));
      bot.mask = kRing - 1;
    }
    uint16_t *dband = dirs + (int64_t)g * G8 * 32;
    const double *dg = diag + g * dstride;
    if (g == 0) {
      TopAnalytic top{ng};
      fin = band_sweep<true, TopAnalytic, Bot3, true>(dg, M, N, M, 0, gap, mismatch, span, top, bot, dband);
    } else if (warp == 0 && crank == 0) {
      TopTagged<false> top{wrap + (gen & 1) * W1, nullptr, (long long)g * W1, M, fmul(ng, (double)(32 * g))};
      fin = band_sweep<true, TopTagged<false>, Bot3, true>(dg, M, N, M, 32 * g, gap, mismatch, span, top, bot, dband);
    } else {
      BigRing *in = &rings[warp];
      TopTagged<true> top{in->slot, &in->cons, (long long)gen * W1, M, fmul(ng, (double)(32 * g))};
      fin = band_sweep<true, TopTagged<true>, Bot3, true>(dg, M, N, M, 32 * g, gap, mismatch, span, top, bot, dband);
      if (lane == 0) in->cons = (long long)(gen + 1) * W1;  // generation done
    }
    if (32 * g + 1 + lane == N) last_val[slot] = fin;
    __syncwarp();
    // (a guard only for launches without the operand layout, never true
    // from abi.cu).  A call site here -- this one, or an empty __noinline__
    // call (-DBIMINE_FAKE_CALL) -- is worth 2.8x on the 4096x4096 sweep:
    // band 0 runs at the same speed either way, but without a call each
    // consumer band's hand-off lag goes from 6.5 to 21.6 us, with the
    // consumer's ring-poll SASS identical (profiles/r2/nw_big_printf_ab.txt).
    // Kept deliberately; tests/test_gpu_perf_guard.py fails if a toolchain
    // change loses it.
#ifndef BIMINE_NO_PRINTF
    if (diag_all == nullptr) printf("bimine: nw_big_kernel band %d without its operand layout\n", g);
#endif
#ifdef BIMINE_FAKE_CALL
    if (diag_all == nullptr) bimine_noop_call(g);
#endif
#ifdef BIMINE_PROF_GLOBAL  // profiling builds: band end times in a device array, no printf call site
    if (lane == 0 && g < 4096) {
      unsigned long long gt;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
      g_prof_band[g] = gt;
    }
#endif
#if defined(BIMINE_NW_PROFILE) || defined(BIMINE_PROF_BAND)
    if (lane == 0) {
      unsigned long long gt;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
      printf("prof band %d cta %d end_ns %llu\n", g, crank, gt);
    }
#endif
  }
  // The kernel ends with the sweep: the traceback is a separate launch
  // (nw_big_traceback_kernel) that reads every CTA's directions after the
  // kernel boundary.  No cluster barrier is needed here either: a CTA's
  // shared memory is last touched remotely by the previous CTA's final ring
  // writes, which its warp 0 has consumed before finishing, and the previous
  // CTA's last remote `cons` poll precedes those writes.
}

// Traceback + threshold filter of large problems (one warp per problem),
// over the 2-bit directions the band pipeline wrote.
template <int MODE>
__device__ void nw_big_traceback_one(const NwArgs &A, const uint32_t *g_dirs_all, const int64_t *dir_off,
                                     const double *last_val, int64_t slot);

template <int MODE>
__global__ void __launch_bounds__(32) nw_big_traceback_kernel(const NwArgs A, const uint32_t *g_dirs_all,
                                                                const int64_t *dir_off, const double *last_val,
                                                                int64_t n_slots) {
  for (int64_t slot = blockIdx.x; slot < n_slots; slot += gridDim.x) nw_big_traceback_one<MODE>(A, g_dirs_all,
                                                                                                dir_off, last_val, slot);
}

template <int MODE>
__device__ void nw_big_traceback_one(const NwArgs &A, const uint32_t *g_dirs_all, const int64_t *dir_off,
                                     const double *last_val, int64_t slot) {
  const int lane = threadIdx.x & 31, warp = 0;
  const int64_t q = A.problem_ids ? A.problem_ids[slot] : slot;
  const int64_t pair = q / A.n_settings;
  const int setting = (int)(q % A.n_settings);
  const int N = A.pair_n[pair], M = A.pair_m[pair];
  const double *__restrict__ sim = A.sim + A.sim_off[pair];
  const int G8 = nw_groups(M);
  const uint16_t *dirs = (const uint16_t *)(g_dirs_all + dir_off[slot]);  // [G][G8][32]
  const double s_last = last_val[slot];
  if (MODE == kNwTable) return;
  // ---- traceback on warp 0: lane 0 walks, the warp stages 16 direction
  // groups (128 steps) of the current band at a time.  A staged cell holds
  // the index step to the next cell of the path in the window's
  // [lane][step] layout (rows of kTbRow bytes): 1 = left (b - 1), kTbRow + 1
  // = up (a - 1: lane - 1, step - 1), kTbRow + 2 = diagonal -- so a step of
  // the walk is one shared-memory byte load and one subtraction.
  if (warp == 0) {
    constexpr int kTbRow = 132;  // 128 steps + 4: lane rows start in distinct banks
    constexpr uint32_t kDelLut = (1u << 16) | ((uint32_t)(kTbRow + 1) << 8) | (uint32_t)(kTbRow + 2);  // by d
    __shared__ __align__(16) uint8_t win[32 * kTbRow];
    __shared__ int win_g, win_k0;
    int a = N, b = M;
    int64_t cnt = 0;
    bimine_match *outm = (MODE == kNwMine) ? A.matches + A.out_off[q] : nullptr;
    uint8_t *st = (MODE == kNwSteps) ? A.steps + A.step_off[q] : nullptr;
    if (lane == 0) {
      win_g = -1;
      win_k0 = 0;
    }
    __syncwarp();
    // a lane's 16 direction words of the window -> its row of step bytes
    auto stage = [&](const uint16_t *w16) {
      uint32_t *row = reinterpret_cast<uint32_t *>(win + lane * kTbRow);
#pragma unroll
      for (int t = 0; t < 16; ++t) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t word = 0;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const uint32_t d = ((uint32_t)w16[t] >> (2 * (4 * h + u))) & 3u;
            word |= ((kDelLut >> (8 * d)) & 0xFFu) << (8 * u);
          }
          row[2 * t + h] = word;
        }
      }
    };
    // the next band's window, loaded into registers while lane 0 walks the
    // current one: the path enters band g-1 at a column no greater than
    // where it entered band g, so the window ending at that column covers
    // any path that moves < ~120 columns left within the band
    uint16_t pre[16];
    int pre_g = -1, pre_k0 = 0;
    while (true) {
      a = __shfl_sync(kFull, a, 0);
      b = __shfl_sync(kFull, b, 0);
      if (!(a > 0 && b > 0)) break;
      const int g = (a - 1) >> 5, l = (a - 1) & 31, k = (b + l - 1) >> 3;
      if (!(g == win_g && k >= win_k0 && k < win_k0 + 16)) {
        if (g == pre_g && k >= pre_k0 && k < pre_k0 + 16) {
          stage(pre);
          __syncwarp();
          if (lane == 0) {
            win_g = g;
            win_k0 = pre_k0;
          }
        } else {
          const int k0 = max(0, k - 15);
          uint16_t cur[16];
#pragma unroll
          for (int t = 0; t < 16; ++t) {
            const int kk = k0 + t;
            cur[t] = kk < G8 ? __ldcg(dirs + ((int64_t)g * G8 + kk) * 32 + lane) : (uint16_t)0;
          }
          stage(cur);
          __syncwarp();
          if (lane == 0) {
            win_g = g;
            win_k0 = k0;
          }
        }
        __syncwarp();
        pre_g = g - 1;  // issue band g-1's loads now; they land during the walk
        if (pre_g >= 0) {
          pre_k0 = max(0, ((b + 30) >> 3) - 15);
#pragma unroll
          for (int t = 0; t < 16; ++t) {
            const int kk = pre_k0 + t;
            pre[t] = kk < G8 ? __ldcg(dirs + ((int64_t)pre_g * G8 + kk) * 32 + lane) : (uint16_t)0;
          }
        }
      }
      if (lane == 0) {
        const int s_base = 8 * win_k0, arow = 32 * win_g + 1;  // window step 0; a = arow + lane
        // the current cell as a window index; valid while the walk stays in
        // the window: each step lowers the lane by <= 1 and the step by <= 2
        int idx = ((a - 1) & 31) * kTbRow + (b + ((a - 1) & 31) - 1 - s_base);
        while (true) {
          const int ll = idx / kTbRow, ss = s_base + idx - ll * kTbRow;
          a = arow + ll;
          b = ss - ll + 1;
          const int safe = min(min(ll, b - 1), (ss - s_base) >> 1);
          auto emit = [&](int del, int ia, int ib) {
            if (MODE == kNwMine) {
              if (del == kTbRow + 2) {
                outm[cnt].i = N - ia;  // score filled below
                outm[cnt].j = M - ib;
                ++cnt;
              }
            } else {
              st[cnt++] = (uint8_t)(del == kTbRow + 2 ? 0 : del == kTbRow + 1 ? 1 : 2);
            }
          };
          if (safe <= 0) {  // the step may leave the window, the band or the table
            const int del = win[idx];
            emit(del, a, b);
            a -= del != 1;
            b -= del != kTbRow + 1;
            break;
          }
#pragma unroll 4
          for (int t = 0; t < safe; ++t) {
            const int del = win[idx];
            if (MODE == kNwMine) {
              if (del == kTbRow + 2) {  // a, b of this cell, off the walk's dependency chain
                const int l2 = idx / kTbRow;
                outm[cnt].i = N - (arow + l2);
                outm[cnt].j = M - (s_base + idx - l2 * kTbRow - l2 + 1);
                ++cnt;
              }
            } else {
              st[cnt++] = (uint8_t)(del == kTbRow + 2 ? 0 : del == kTbRow + 1 ? 1 : 2);
            }
            idx -= del;
          }
        }
      }
      __syncwarp();
    }
    cnt = __shfl_sync(kFull, cnt, 0);
    if (MODE == kNwSteps) {
      if (lane == 0) {
        while (a > 0) {
          st[cnt++] = 1u;
          --a;
        }
        while (b > 0) {
          st[cnt++] = 2u;
          --b;
        }
        A.n_steps[q] = (int32_t)cnt;
      }
    } else {
      // gather the scores in parallel, keep those at or above the threshold:
      // 8 batches of 32 matches per round, all their loads in flight before
      // the in-order compaction (the scores are scattered over the whole
      // N x M matrix: one round trip per batch made this half the traceback)
      const double thr = nw_threshold(A, setting);
      int64_t kept = 0;
      constexpr int kRounds = 8;
      for (int64_t base = 0; base < cnt; base += 32 * kRounds) {
        int32_t ii[kRounds], jj[kRounds];
        double vv[kRounds];
#pragma unroll
        for (int r = 0; r < kRounds; ++r) {
          const int64_t c = base + 32 * r + lane;
          ii[r] = 0;
          jj[r] = 0;
          if (c < cnt) {
            ii[r] = outm[c].i;
            jj[r] = outm[c].j;
          }
        }
#pragma unroll
        for (int r = 0; r < kRounds; ++r) {
          const int64_t c = base + 32 * r + lane;
          vv[r] = c < cnt ? sim[(int64_t)ii[r] * M + jj[r]] : 0.0;
        }
        __syncwarp();  // every read of this round's entries before any write
#pragma unroll
        for (int r = 0; r < kRounds; ++r) {
          const int64_t c = base + 32 * r + lane;
          const bool keep = c < cnt && vv[r] >= thr;
          const unsigned bal = __ballot_sync(kFull, keep);
          if (keep) {
            bimine_match &o = outm[kept + __popc(bal & ((1u << lane) - 1u))];
            o.score = vv[r];
            o.i = ii[r];
            o.j = jj[r];
          }
          kept += __popc(bal);
        }
        __syncwarp();
      }
      if (lane == 0) A.counts[q] = (int32_t)kept;
    }
    if (lane == 0 && A.score) A.score[q] = s_last;
#if defined(BIMINE_NW_PROFILE) || defined(BIMINE_PROF_TB)
    if (lane == 0) {
      unsigned long long gt;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
      printf("prof traceback end_ns %llu\n", gt);
    }
#endif
  }
}

}  // namespace bimine
