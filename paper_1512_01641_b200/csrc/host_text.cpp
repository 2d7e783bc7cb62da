// host_text.cpp -- native host side of the boundary: the tokenizer and the
// joint vocabulary.
//
// tokenize (text.py:97-104) is `[t.strip(string.punctuation) for t in
// text.lower().split() if ...]`.  For ASCII text that is exactly:
// lowercase A-Z, split on runs of the ASCII characters str.isspace()
// accepts (\t \n \v \f \r \x1c-\x1f and space), strip the 32 ASCII
// punctuation characters from both ends, drop empty tokens.  Text whose
// code points are all below U+0180 (Latin-1 Supplement, Latin Extended-A:
// Polish, German, French, ...) is handled natively too: there str.lower()
// is the one-to-one map of lower_latin() (except U+0130, which lowers to
// two code points) and str.isspace() adds U+0085 and U+00A0.  Any other
// sentence is reported back (length -1) and tokenised by the Python rules
// on the host, through the same vocabulary, so every path gives the same
// ids.
//
// The vocabulary is a flat open-addressing table (32-byte slots: hash,
// id, length, the first 16 bytes of the word; all word bytes in a block
// arena, so bimine_vocab_word pointers stay valid).  A large batch is tokenised in three phases: (1) threads
// split, lowercase, hash and LOOK UP their contiguous sentence range in
// the read-only table, recording words not found; (2) one thread inserts
// the missing words in batch order -- thread ranges are in sentence order,
// so ids are assigned in first-occurrence order exactly as a serial pass
// would; (3) threads patch the new ids in, count distinct tokens per
// sentence and copy their tokens to the output.
#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <chrono>
#include <cstdio>
#include <thread>
#include <mutex>
#include <new>
#include <utility>
#include <vector>

#include <emmintrin.h>
#include <sys/mman.h>

#include "../../include/bimine_b200.h"

namespace {

inline uint64_t hash_words(const char *p, uint32_t n) {
  // p is readable and zero-padded up to the next multiple of 8 bytes.
  uint64_t h = 0x243F6A8885A308D3ull ^ ((uint64_t)n * 0x9E3779B97F4A7C15ull);
  for (uint32_t i = 0; i < n; i += 8) {
    uint64_t w;
    memcpy(&w, p + i, 8);
    h = (h ^ w) * 0xBF58476D1CE4E5B9ull;
    h ^= h >> 31;
  }
  h ^= h >> 30;
  h *= 0x94D049BB133111EBull;
  return h ^ (h >> 29);
}

// zero-padded copy of a word (the layout find() and hash_words() read)
inline const char *padded(const char *w, uint32_t n, std::vector<char> &pad) {
  if (pad.size() < (size_t)n + 16) pad.resize((size_t)n + 16);
  memcpy(pad.data(), w, n);
  memset(pad.data() + n, 0, 16);
  return pad.data();
}

// str.lower() of a code point below U+0180 other than U+0130 (checked
// exhaustively against CPython in tests/test_host.py)
constexpr uint32_t lower_latin(uint32_t c) {
  if (c < 0x80) return (c - 'A' < 26u) ? c + 32 : c;
  if (c >= 0xC0 && c <= 0xDE && c != 0xD7) return c + 32;
  if (c >= 0x100 && c <= 0x137) return (c & 1) ? c : c + 1;
  if (c >= 0x139 && c <= 0x148) return (c & 1) ? c + 1 : c;
  if (c >= 0x14A && c <= 0x177) return (c & 1) ? c : c + 1;
  if (c == 0x178) return 0xFF;
  if (c >= 0x179 && c <= 0x17E) return (c & 1) ? c + 1 : c;
  return c;
}

// A non-ASCII sentence of code points < U+0180 (not U+0130): lowered, as
// UTF-8, into `out`, whitespace code points as ' '; returns its code-point
// count, or -1 when the sentence needs the Python rules.
int64_t lower_latin_sentence(const unsigned char *p, int64_t L, std::vector<unsigned char> &out) {
  out.clear();
  int64_t cps = 0;
  for (int64_t x = 0; x < L; ++cps) {
    const unsigned char b = p[x];
    uint32_t c;
    if (b < 0x80) {
      c = b;
      x += 1;
    } else if ((b & 0xE0) == 0xC0 && x + 1 < L && (p[x + 1] & 0xC0) == 0x80) {
      c = ((uint32_t)(b & 0x1F) << 6) | (p[x + 1] & 0x3F);
      if (c < 0x80 || c >= 0x180 || c == 0x130) return -1;  // overlong, or outside the table
      x += 2;
    } else {
      return -1;
    }
    if (c == 0x85 || c == 0xA0) {
      out.push_back(' ');
      continue;
    }
    c = lower_latin(c);
    if (c < 0x80) {
      out.push_back((unsigned char)c);
    } else {
      out.push_back((unsigned char)(0xC0 | (c >> 6)));
      out.push_back((unsigned char)(0x80 | (c & 0x3F)));
    }
  }
  return cps;
}

constexpr bool is_space(unsigned char c) {
  return c == ' ' || (c >= '\t' && c <= '\r') || (c >= 0x1c && c <= 0x1f);
}

// byte classes of the split: 1 = whitespace, 2 = punctuation
struct ByteClass {
  uint8_t c[256] = {};
  constexpr ByteClass() {
    const char *P = "!\"#$%&'()*+,-./:;<=>?@[\\]^_`{|}~";
    for (int i = 0; P[i]; ++i) c[(unsigned char)P[i]] = 2;
    for (int i = 0; i < 256; ++i)
      if (is_space((unsigned char)i)) c[i] = 1;
  }
};
constexpr ByteClass kClass;

// A-Z -> a-z in each byte of w (other bytes, UTF-8 included, unchanged)
inline uint64_t lower8(uint64_t w) {
  const uint64_t h = w & 0x7F7F7F7F7F7F7F7Full;
  const uint64_t ge_a = h + 0x3F3F3F3F3F3F3F3Full;  // high bit: >= 'A'
  const uint64_t gt_z = h + 0x2525252525252525ull;  // high bit: > 'Z'
  return w | (((ge_a ^ gt_z) & ~w & 0x8080808080808080ull) >> 2);
}

// the low n bytes of w (n in 0..8)
inline uint64_t low_bytes(uint64_t w, uint32_t n) { return n >= 8 ? w : w & ((1ull << (8 * n)) - 1); }

// hash_words of a word of n <= 16 bytes given as its two zero-padded words
inline uint64_t hash_keys(uint64_t k0, uint64_t k1, uint32_t n) {
  uint64_t h = 0x243F6A8885A308D3ull ^ ((uint64_t)n * 0x9E3779B97F4A7C15ull);
  if (n > 0) {
    h = (h ^ k0) * 0xBF58476D1CE4E5B9ull;
    h ^= h >> 31;
  }
  if (n > 8) {
    h = (h ^ k1) * 0xBF58476D1CE4E5B9ull;
    h ^= h >> 31;
  }
  h ^= h >> 30;
  h *= 0x94D049BB133111EBull;
  return h ^ (h >> 29);
}

struct PunctTable {
  bool p[256] = {};
  constexpr PunctTable() {
    const char *P = "!\"#$%&'()*+,-./:;<=>?@[\\]^_`{|}~";
    for (int i = 0; P[i]; ++i) p[(unsigned char)P[i]] = true;
  }
};
constexpr PunctTable kPunct;

int host_threads() {
  static const int n = [] {
    const char *e = getenv("BIMINE_HOST_THREADS");
    int v = e ? atoi(e) : (int)std::thread::hardware_concurrency();
    return std::max(1, std::min(v, 64));
  }();
  return n;
}

// Phase 1 state of one thread: its sentences [k0, k1).
struct TokRange {
  int64_t k0 = 0, k1 = 0;
  std::vector<int32_t> tok;  // id, or -(index into miss) - 1
  struct Miss {
    uint64_t hash;
    uint32_t off, len;  // in `words`
  };
  std::vector<Miss> miss;
  std::vector<char> words;  // lowercased missing words, zero-padded like tokenize_range's
  std::vector<int32_t> resolved;
  int64_t out_off = 0;
  void reset(int64_t a, int64_t b) {  // (buffers keep their capacity from call to call)
    k0 = a;
    k1 = b;
    tok.clear();
    miss.clear();
    words.clear();
    resolved.clear();
    out_off = 0;
  }
};

}  // namespace

struct bimine_vocab {
  // the batch tokenizer's per-thread state, kept between calls (no fresh
  // pages to fault in per call); one tokenisation at a time per vocabulary
  std::mutex tok_mu;
  std::vector<TokRange> tok_ranges;
  struct Slot {
    uint64_t hash;
    int32_t id;  // -1: empty
    uint32_t len;
    uint64_t key[2];  // first 16 bytes of the word, zero-padded
  };
  // the slot array, 2 MB aligned and on transparent huge pages where the
  // kernel allows: lookups are random over tens of MB, and with 4 KB pages
  // nearly every one also missed the TLB
  struct Slots {
    Slot *p = nullptr;
    size_t n = 0;
    explicit Slots(size_t count) : n(count) {
      const size_t bytes = ((count * sizeof(Slot)) + (2u << 20) - 1) & ~(size_t)((2u << 20) - 1);
      p = static_cast<Slot *>(aligned_alloc(2u << 20, bytes));
      if (!p) throw std::bad_alloc();
#ifdef MADV_HUGEPAGE
      madvise(p, bytes, MADV_HUGEPAGE);
#endif
      for (size_t i = 0; i < count; ++i) p[i] = Slot{0, -1, 0, {0, 0}};
    }
    Slots(const Slots &) = delete;
    Slots &operator=(const Slots &) = delete;
    ~Slots() { free(p); }
    void swap(Slots &o) {
      std::swap(p, o.p);
      std::swap(n, o.n);
    }
    size_t size() const { return n; }
    Slot &operator[](size_t i) { return p[i]; }
    const Slot &operator[](size_t i) const { return p[i]; }
    const Slot *begin() const { return p; }
    const Slot *end() const { return p + n; }
  };
  Slots slots{1u << 16};
  size_t mask = (1u << 16) - 1;
  std::vector<const char *> word_ptr;  // id -> bytes in `blocks`
  std::vector<uint32_t> word_len;
  std::vector<std::unique_ptr<char[]>> blocks;
  size_t block_used = 0, block_cap = 0;

  int32_t size() const { return (int32_t)word_ptr.size(); }

  const Slot *slot_of(uint64_t h) const { return &slots[h & mask]; }

  // w: n bytes, then zeros to at least max(16, n rounded up to 8) bytes
  int32_t find(uint64_t h, const char *w, uint32_t n) const {
    uint64_t k0, k1;
    memcpy(&k0, w, 8);
    memcpy(&k1, w + 8, 8);
    return find_keys(h, k0, k1, n, w);
  }

  // k0, k1: the word's first 16 bytes, zero-padded; w: the whole word
  // (read only beyond byte 16)
  int32_t find_keys(uint64_t h, uint64_t k0, uint64_t k1, uint32_t n, const char *w) const {
    for (size_t i = h & mask;; i = (i + 1) & mask) {
      const Slot &s = slots[i];
      if (s.id < 0) return -1;
      if (s.hash == h && s.len == n && s.key[0] == k0 && s.key[1] == k1 &&
          (n <= 16 || memcmp(word_ptr[s.id] + 16, w + 16, n - 16) == 0))
        return s.id;
    }
  }

  int32_t insert(uint64_t h, const char *w, uint32_t n) {  // w absent
    if (block_used + n + 1 > block_cap) {
      block_cap = std::max<size_t>(1u << 20, (size_t)n + 1);
      blocks.emplace_back(new char[block_cap]);
      block_used = 0;
    }
    char *dst = blocks.back().get() + block_used;
    memcpy(dst, w, n);
    dst[n] = 0;
    block_used += n + 1;
    const int32_t id = size();
    word_ptr.push_back(dst);
    word_len.push_back(n);
    if ((size_t)(id + 1) * 2 > slots.size()) grow();
    size_t i = h & mask;
    while (slots[i].id >= 0) i = (i + 1) & mask;
    Slot &s = slots[i];
    s = Slot{h, id, n, {0, 0}};
    memcpy(s.key, w, std::min<uint32_t>(n, 16));
    return id;
  }

  void grow() {
    Slots old(slots.size() * 2);
    old.swap(slots);
    mask = slots.size() - 1;
    for (const Slot &s : old)
      if (s.id >= 0) {
        size_t i = s.hash & mask;
        while (slots[i].id >= 0) i = (i + 1) & mask;
        slots[i] = s;
      }
  }

  int32_t get(uint64_t h, const char *w, uint32_t n) {
    const int32_t id = find(h, w, n);
    return id >= 0 ? id : insert(h, w, n);
  }
};

namespace {

// Per sentence, two passes: split + lowercase + hash every token and
// prefetch its home slot, then resolve them (the table is far larger than
// the caches; the prefetches overlap the misses).
// Sentences as one buffer + offsets, or as one pointer + length each.
struct BufSentences {
  const unsigned char *buf;
  const int64_t *off;
  const unsigned char *ptr(int64_t k) const { return buf + off[k]; }
  int64_t len(int64_t k) const { return off[k + 1] - off[k]; }
};
struct PtrSentences {
  const unsigned char *const *p;
  const int64_t *n;
  const unsigned char *ptr(int64_t k) const { return p[k]; }
  int64_t len(int64_t k) const { return n[k]; }
};

// Whitespace bitmap of p[0, L): bit x of sp[x / 64] set when p[x] is
// whitespace or x >= L (up to the end of the last word); returns false if
// a byte is >= 0x80.  SSE2, 16 bytes per step.
inline bool space_bitmap(const unsigned char *p, int64_t L, std::vector<uint64_t> &sp) {
  const size_t nw = (size_t)(L >> 6) + 1;
  if (sp.size() < nw) sp.resize(nw);
  const __m128i c32 = _mm_set1_epi8(32), c9 = _mm_set1_epi8(9), c4 = _mm_set1_epi8(4), c28 = _mm_set1_epi8(28),
                c3 = _mm_set1_epi8(3);
  uint32_t hi = 0;
  for (size_t w = 0; w < nw; ++w) {
    uint64_t m = 0;
    for (int q = 0; q < 4; ++q) {
      const int64_t x = (int64_t)(w * 64 + q * 16);
      __m128i v;
      uint32_t tail = 0;  // positions >= L
      if (x + 16 <= L) {
        v = _mm_loadu_si128(reinterpret_cast<const __m128i *>(p + x));
      } else {
        alignas(16) unsigned char t[16] = {};
        if (x < L) memcpy(t, p + x, (size_t)(L - x));
        v = _mm_load_si128(reinterpret_cast<const __m128i *>(t));
        tail = x >= L ? 0xFFFFu : (0xFFFFu << (L - x)) & 0xFFFFu;
      }
      hi |= (uint32_t)_mm_movemask_epi8(v);
      const __m128i t1 = _mm_sub_epi8(v, c9), t2 = _mm_sub_epi8(v, c28);
      const __m128i sp16 = _mm_or_si128(_mm_cmpeq_epi8(v, c32),
                                        _mm_or_si128(_mm_cmpeq_epi8(_mm_min_epu8(t1, c4), t1),
                                                     _mm_cmpeq_epi8(_mm_min_epu8(t2, c3), t2)));
      m |= (uint64_t)(((uint32_t)_mm_movemask_epi8(sp16) | tail) & 0xFFFFu) << (q * 16);
    }
    sp[w] = m;
  }
  return hi == 0;
}

// first x' >= x whose bit in sp equals `want` (a bit past L is always set)
inline int64_t next_bit(const uint64_t *sp, int64_t x, bool want) {
  size_t w = (size_t)(x >> 6);
  uint64_t m = (want ? sp[w] : ~sp[w]) & (~0ull << (x & 63));
  while (!m) {
    ++w;
    m = want ? sp[w] : ~sp[w];
  }
  return (int64_t)(w * 64) + __builtin_ctzll(m);
}

template <class Sent>
void tokenize_range(const bimine_vocab &v, const Sent &sent, TokRange &r, int32_t *len_out, int32_t *chars_out) {
  // a token: its hash and first 16 bytes (lowered, zero-padded); a word
  // longer than 16 bytes also has a lowered, padded copy in `low`
  struct Tok {
    uint64_t hash, k0, k1;
    uint32_t len, off;
  };
  // two sentences in flight: sentence k is split (its vocabulary slots
  // prefetched) before sentence k - 1's tokens are looked up
  std::vector<Tok> toks[2];
  std::vector<char> low[2];
  std::vector<unsigned char> lat;  // a Latin sentence, lowered
  std::vector<uint64_t> sp;
  {
    int64_t bytes = 0;
    for (int64_t k = r.k0; k < r.k1; ++k) bytes += sent.len(k);
    r.tok.reserve((size_t)(bytes / 4 + (r.k1 - r.k0)));
  }
  auto resolve = [&](int64_t k, int par) {
    const std::vector<Tok> &tk = toks[par];
    for (const Tok &t : tk) {
      const char *lw = t.len > 16 ? low[par].data() + t.off : nullptr;
      int32_t id = v.find_keys(t.hash, t.k0, t.k1, t.len, lw);
      if (id < 0) {  // the padded word for the insert phase
        const uint32_t wo = (uint32_t)r.words.size(), padn = ((t.len + 7) & ~7u) + 16;
        r.words.resize(wo + padn, 0);
        char *w = r.words.data() + wo;
        if (lw) {
          memcpy(w, lw, padn);
        } else {
          memcpy(w, &t.k0, 8);
          memcpy(w + 8, &t.k1, 8);
        }
        r.miss.push_back({t.hash, wo, t.len});
        id = -(int32_t)r.miss.size();
      }
      r.tok.push_back(id);
    }
    len_out[k] = (int32_t)tk.size();
  };
  int64_t pending = -1;  // sentence whose tokens await lookup, in toks[cur ^ 1]
  int cur = 0;
  for (int64_t k = r.k0; k < r.k1; ++k) {
    const unsigned char *p = sent.ptr(k);
    int64_t L = sent.len(k);
    chars_out[k] = (int32_t)L;
    if (!space_bitmap(p, L, sp)) {
      const int64_t cps = lower_latin_sentence(p, L, lat);
      if (cps < 0) {
        len_out[k] = -1;  // the caller applies the Unicode rules
        continue;
      }
      chars_out[k] = (int32_t)cps;  // len(text): code points
      p = lat.data();
      L = (int64_t)lat.size();
      space_bitmap(p, L, sp);  // (whitespace is ASCII after lowering)
    }
    std::vector<Tok> &tk = toks[cur];
    std::vector<char> &lo = low[cur];
    tk.clear();
    lo.clear();
    for (int64_t x = next_bit(sp.data(), 0, false); x < L; x = next_bit(sp.data(), x, false)) {
      int64_t a = x;
      x = next_bit(sp.data(), x, true);
      int64_t b = x;
      while (a < b && kClass.c[p[a]] == 2) ++a;
      while (b > a && kClass.c[p[b - 1]] == 2) --b;
      if (b == a) continue;
      const uint32_t n = (uint32_t)(b - a);
      uint64_t k0, k1;
      if (a + 16 <= L) {
        memcpy(&k0, p + a, 8);
        memcpy(&k1, p + a + 8, 8);
      } else {
        unsigned char t[16] = {};
        memcpy(t, p + a, (size_t)std::min<int64_t>(16, L - a));
        memcpy(&k0, t, 8);
        memcpy(&k1, t + 8, 8);
      }
      k0 = lower8(low_bytes(k0, n));
      k1 = n > 8 ? lower8(low_bytes(k1, n - 8)) : 0;
      Tok t{0, k0, k1, n, 0};
      if (n <= 16) {
        t.hash = hash_keys(k0, k1, n);
      } else {  // a long word: lowered, padded copy
        t.off = (uint32_t)lo.size();
        lo.resize(lo.size() + ((n + 7) & ~7u) + 16, 0);
        char *w = lo.data() + t.off;
        for (uint32_t i = 0; i < n; ++i) {
          const unsigned char c = p[a + i];
          w[i] = (char)((unsigned)(c - 'A') < 26u ? c | 0x20 : c);
        }
        t.hash = hash_words(w, n);
      }
      __builtin_prefetch(v.slot_of(t.hash));
      tk.push_back(t);
    }
    if (pending >= 0) resolve(pending, cur ^ 1);
    pending = k;
    cur ^= 1;
  }
  if (pending >= 0) resolve(pending, cur ^ 1);
}

// ids, and distinct ids per sentence by a per-thread stamp per id
void finish_range(TokRange &r, const int32_t *len_out, int32_t *uniq_out, int32_t *tokens, int32_t n_ids) {
  int32_t *dst = tokens + r.out_off;
  const int32_t *src = r.tok.data();
  std::vector<uint32_t> stamp((size_t)std::max(n_ids, 1), 0u);
  uint32_t tag = 0;
  for (int64_t k = r.k0; k < r.k1; ++k) {
    const int32_t n = len_out[k];
    if (n < 0) {
      uniq_out[k] = 0;
      continue;
    }
    ++tag;
    int32_t u = 0;
    for (int32_t i = 0; i < n; ++i) {
      const int32_t id = src[i] >= 0 ? src[i] : r.resolved[-src[i] - 1];
      dst[i] = id;
      if (stamp[id] != tag) {
        stamp[id] = tag;
        ++u;
      }
    }
    uniq_out[k] = u;
    dst += n;
    src += n;
  }
}

}  // namespace

extern "C" {

int bimine_vocab_create(bimine_vocab **out) {
  if (!out) return BIMINE_E_ARG;
  *out = new bimine_vocab();
  return BIMINE_OK;
}

int bimine_vocab_destroy(bimine_vocab *v) {
  delete v;
  return BIMINE_OK;
}

int64_t bimine_vocab_size(const bimine_vocab *v) { return v ? (int64_t)v->size() : -1; }

int bimine_vocab_add_batch(bimine_vocab *v, const char *buf, const int64_t *off, int64_t n, int32_t *ids) {
  if (!v || (n > 0 && (!buf || !off || !ids))) return BIMINE_E_ARG;
  std::vector<char> pad;
  for (int64_t k = 0; k < n; ++k) {
    const uint32_t len = (uint32_t)(off[k + 1] - off[k]);
    const char *w = padded(buf + off[k], len, pad);
    ids[k] = v->get(hash_words(w, len), w, len);
  }
  return BIMINE_OK;
}

int bimine_vocab_word(const bimine_vocab *v, int32_t id, const char **ptr, int64_t *len) {
  if (!v || !ptr || !len || id < 0 || id >= v->size()) return BIMINE_E_ARG;
  *ptr = v->word_ptr[id];
  *len = (int64_t)v->word_len[id];
  return BIMINE_OK;
}

}  // extern "C"

namespace {

// The three phases over `n` sentences split into ranges of about `bytes_of`
// bytes each (>= 256 KB per thread).
template <class Sent, class Prefix>
int tokenize_sentences(bimine_vocab *v, const Sent &sent, int64_t n, Prefix prefix_bytes, int32_t *tokens,
                       int64_t cap, int64_t *n_tokens, int32_t *len_out, int32_t *uniq_out, int32_t *chars_out) {
  *n_tokens = 0;
  if (n <= 0) return BIMINE_OK;
  const int64_t bytes = prefix_bytes(n);
  const int nt = (int)std::max<int64_t>(1, std::min<int64_t>(host_threads(), bytes >> 18));
  std::lock_guard<std::mutex> lk(v->tok_mu);
  std::vector<TokRange> &R = v->tok_ranges;
  if ((int)R.size() < nt) R.resize(nt);
  for (int t = 0; t < nt; ++t) {
    const int64_t k0 = t == 0 ? 0 : R[t - 1].k1;
    int64_t k1 = n;
    if (t < nt - 1) {  // first sentence whose byte prefix reaches the thread's share
      int64_t lo = k0, hi = n;
      const int64_t want = bytes * (t + 1) / nt;
      while (lo < hi) {
        const int64_t mid = (lo + hi) / 2;
        if (prefix_bytes(mid) < want) lo = mid + 1;
        else hi = mid;
      }
      k1 = lo;
    }
    R[t].reset(k0, k1);
  }
  auto parallel = [&](auto &&fn) {
    if (nt == 1) return fn(R[0]);
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t) pool.emplace_back([&, t] { fn(R[t]); });
    fn(R[0]);
    for (auto &th : pool) th.join();
  };
#ifdef BIMINE_TOK_PROFILE
  auto clk = [] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
  const double c0 = clk();
#endif
  parallel([&](TokRange &r) { tokenize_range(*v, sent, r, len_out, chars_out); });
#ifdef BIMINE_TOK_PROFILE
  const double c1 = clk();
#endif
  int64_t total = 0;
  for (int t = 0; t < nt; ++t) {
    R[t].out_off = total;
    total += (int64_t)R[t].tok.size();
  }
  if (total > cap) return BIMINE_E_LIMIT;  // vocabulary unchanged
  for (int t = 0; t < nt; ++t) {  // serial: first-occurrence id order
    TokRange &r = R[t];
    r.resolved.resize(r.miss.size());
    for (size_t i = 0; i < r.miss.size(); ++i)
      r.resolved[i] = v->get(r.miss[i].hash, r.words.data() + r.miss[i].off, r.miss[i].len);
  }
#ifdef BIMINE_TOK_PROFILE
  const double c2 = clk();
#endif
  const int32_t n_ids = v->size();
  parallel([&](TokRange &r) { finish_range(r, len_out, uniq_out, tokens, n_ids); });
#ifdef BIMINE_TOK_PROFILE
  fprintf(stderr, "tokenize: %d threads, split %.1f ms, insert %.1f ms, finish %.1f ms\n", nt, c1 - c0, c2 - c1, clk() - c2);
#endif
  *n_tokens = total;
  return BIMINE_OK;
}

}  // namespace

extern "C" {

int bimine_tokenize_batch(bimine_vocab *v, const char *buf, const int64_t *off, int64_t n, int32_t *tokens,
                          int64_t cap, int64_t *n_tokens, int32_t *len_out, int32_t *uniq_out, int32_t *chars_out) {
  if (!v || !n_tokens || (n > 0 && (!buf || !off || !len_out || !uniq_out || !chars_out)))
    return BIMINE_E_ARG;
  const BufSentences sent{(const unsigned char *)buf, off};
  return tokenize_sentences(v, sent, n, [&](int64_t k) { return off[k] - off[0]; }, tokens, cap, n_tokens, len_out,
                            uniq_out, chars_out);
}

int bimine_tokenize_ptrs(bimine_vocab *v, const char *const *ptrs, const int64_t *lens, int64_t n,
                         const int64_t *len_prefix, int32_t *tokens, int64_t cap, int64_t *n_tokens,
                         int32_t *len_out, int32_t *uniq_out, int32_t *chars_out) {
  if (!v || !n_tokens || (n > 0 && (!ptrs || !lens || !len_prefix || !len_out || !uniq_out || !chars_out)))
    return BIMINE_E_ARG;
  const PtrSentences sent{(const unsigned char *const *)ptrs, lens};
  return tokenize_sentences(v, sent, n, [&](int64_t k) { return len_prefix[k]; }, tokens, cap, n_tokens, len_out,
                            uniq_out, chars_out);
}

}  // extern "C"
