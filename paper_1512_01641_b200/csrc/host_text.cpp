// host_text.cpp -- native host side of the boundary: the tokenizer and the
// joint vocabulary.
//
// tokenize (text.py:97-104) is `[t.strip(string.punctuation) for t in
// text.lower().split() if ...]`.  For ASCII text that is exactly:
// lowercase A-Z, split on runs of the ASCII characters str.isspace()
// accepts (\t \n \v \f \r \x1c-\x1f and space), strip the 32 ASCII
// punctuation characters from both ends, drop empty tokens.  A sentence
// with any non-ASCII byte is reported back (length -1) and tokenised by
// the Python rules on the host (full Unicode lower()/split()), through the
// same vocabulary, so both paths produce the same ids.
#include <cstdint>
#include <cstring>
#include <string>
#include <string_view>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "../../include/bimine_b200.h"

struct bimine_vocab {
  std::unordered_map<std::string, int32_t> ids;
  std::vector<const std::string *> words;  // id -> key stored in `ids`

  int32_t get(std::string_view w) {
    auto it = ids.find(std::string(w));
    if (it != ids.end()) return it->second;
    const int32_t id = (int32_t)words.size();
    auto ins = ids.emplace(std::string(w), id);
    words.push_back(&ins.first->first);
    return id;
  }
};

namespace {

constexpr bool is_space(unsigned char c) {
  return c == ' ' || (c >= '\t' && c <= '\r') || (c >= 0x1c && c <= 0x1f);
}

bool is_punct(unsigned char c) {
  static const char *P = "!\"#$%&'()*+,-./:;<=>?@[\\]^_`{|}~";
  return c < 128 && c && strchr(P, c) != nullptr;
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

int64_t bimine_vocab_size(const bimine_vocab *v) { return v ? (int64_t)v->words.size() : -1; }

int bimine_vocab_add_batch(bimine_vocab *v, const char *buf, const int64_t *off, int64_t n, int32_t *ids) {
  if (!v || (n > 0 && (!buf || !off || !ids))) return BIMINE_E_ARG;
  for (int64_t k = 0; k < n; ++k) ids[k] = v->get(std::string_view(buf + off[k], (size_t)(off[k + 1] - off[k])));
  return BIMINE_OK;
}

int bimine_vocab_word(const bimine_vocab *v, int32_t id, const char **ptr, int64_t *len) {
  if (!v || !ptr || !len || id < 0 || id >= (int32_t)v->words.size()) return BIMINE_E_ARG;
  *ptr = v->words[id]->data();
  *len = (int64_t)v->words[id]->size();
  return BIMINE_OK;
}

int bimine_tokenize_batch(bimine_vocab *v, const char *buf, const int64_t *off, int64_t n, int32_t *tokens,
                          int64_t cap, int64_t *n_tokens, int32_t *len_out, int32_t *uniq_out, int32_t *chars_out) {
  if (!v || !n_tokens || (n > 0 && (!buf || !off || !len_out || !uniq_out || !chars_out)))
    return BIMINE_E_ARG;
  int64_t t = 0;
  std::string low;
  std::unordered_set<int32_t> seen;
  for (int64_t k = 0; k < n; ++k) {
    const unsigned char *p = (const unsigned char *)buf + off[k];
    const int64_t L = off[k + 1] - off[k];
    bool ascii = true;
    for (int64_t x = 0; x < L; ++x)
      if (p[x] >= 0x80) {
        ascii = false;
        break;
      }
    chars_out[k] = (int32_t)L;
    if (!ascii) {
      len_out[k] = -1;  // the caller applies the Unicode rules
      uniq_out[k] = 0;
      continue;
    }
    const int64_t t0 = t;
    seen.clear();
    int64_t x = 0;
    while (x < L) {
      while (x < L && is_space(p[x])) ++x;
      int64_t a = x;
      while (x < L && !is_space(p[x])) ++x;
      int64_t b = x;
      while (a < b && is_punct(p[a])) ++a;
      while (b > a && is_punct(p[b - 1])) --b;
      if (b > a) {
        low.assign((const char *)p + a, (size_t)(b - a));
        for (char &c : low)
          if (c >= 'A' && c <= 'Z') c = (char)(c - 'A' + 'a');
        if (t >= cap) return BIMINE_E_LIMIT;
        const int32_t id = v->get(low);
        tokens[t++] = id;
        seen.insert(id);
      }
    }
    len_out[k] = (int32_t)(t - t0);
    uniq_out[k] = (int32_t)seen.size();
  }
  *n_tokens = t;
  return BIMINE_OK;
}

}  // extern "C"
