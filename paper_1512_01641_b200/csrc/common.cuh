// common.cuh -- shared device helpers for the bimine B200 kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/bimine_b200.h"
#include "glibc_exp.cuh"

namespace bimine {

constexpr unsigned kFull = 0xffffffffu;

// Token ids as int32, or packed little-endian in 3 bytes each
// (bimine_batch.token_bytes == 3): tokens[k] reads either (one uniform
// branch per load).
struct TokenView {
  const int32_t *t32;
  bool packed;
  __device__ __forceinline__ int32_t operator[](int64_t k) const {
    if (packed) {
      const uint8_t *q = reinterpret_cast<const uint8_t *>(t32) + 3 * k;
      return (int32_t)((uint32_t)__ldg(q) | ((uint32_t)__ldg(q + 1) << 8) | ((uint32_t)__ldg(q + 2) << 16));
    }
    return t32[k];
  }
};

// The same with the width fixed at compile time (kernels instantiated per form).
template <bool kPacked>
struct TokenViewT {
  const int32_t *t32;
  __device__ __forceinline__ int32_t operator[](int64_t k) const {
    if (kPacked) {
      const uint8_t *q = reinterpret_cast<const uint8_t *>(t32) + 3 * k;
      return (int32_t)((uint32_t)__ldg(q) | ((uint32_t)__ldg(q + 1) << 8) | ((uint32_t)__ldg(q + 2) << 16));
    }
    return t32[k];
  }
};

// Device-side copy of the batch descriptor (all device pointers).
struct BatchDev {
  TokenView tokens;
  const int64_t *sent_tok_off;
  const int32_t *sent_len;
  const int32_t *sent_uniq;
  const int32_t *sent_chars;
  const int64_t *pair_src;
  const int32_t *pair_n;
  const int64_t *pair_tgt;
  const int32_t *pair_m;
  const int64_t *pair_sim_off;
  int64_t n_pairs;
};

// One dictionary entry as the score kernel reads it: p and the target id
// in one 16-byte record (one load per walked entry).
struct __align__(16) DictEntry {
  double p;
  int32_t t;
  int32_t pad;
};

struct DictDev {
  int64_t n_rows;
  const int64_t *row_ptr;
  const int32_t *tgt;
  const double *prob;
  // the same CSR for the score kernel: row s = entries [rowdesc[s] >> 24,
  // (rowdesc[s] >> 24) + (rowdesc[s] & 0xFFFFFF)) of `ent`
  const uint64_t *rowdesc;
  const DictEntry *ent;
};

struct Model {
  double w[6];
  double bias, a, b;
  double mean[6];
  double scale[6];
};

inline BatchDev to_dev(const bimine_batch &b) {
  return BatchDev{TokenView{b.tokens, b.token_bytes == 3}, b.sent_tok_off, b.sent_len, b.sent_uniq, b.sent_chars,
                  b.pair_src, b.pair_n, b.pair_tgt, b.pair_m, b.pair_sim_off, b.n_pairs};
}

inline Model to_model(const double *v) {
  Model m;
  for (int k = 0; k < 6; ++k) m.w[k] = v[k];
  m.bias = v[6];
  m.a = v[7];
  m.b = v[8];
  for (int k = 0; k < 6; ++k) m.mean[k] = v[9 + k];
  for (int k = 0; k < 6; ++k) m.scale[k] = v[15 + k];
  return m;
}

// Multiplicative (Fibonacci) hashing: the top `bits` bits of key * phi.
__device__ __forceinline__ uint32_t hash_slot(int32_t key, int shift) {
  return ((uint32_t)key * 0x9E3779B1u) >> shift;
}

// The exp table as a device global (the score kernel stages it in smem).
__device__ const uint64_t kExpTableDev[256] = {
#include "exp_table.inc"
};

}  // namespace bimine
