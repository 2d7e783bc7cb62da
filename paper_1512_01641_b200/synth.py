"""Seeded synthetic comparable corpora in the shapes of BASELINE.json.

One generator emits, from one seed, both the packed integer form the
GPU consumes and (on demand) the exact sentence strings the reference
consumes, so the same inputs drive the CUDA path and the CPU oracle.
The recipe is SURVEY.md section 8(d), generalising the reference's test
fixture `make_mining_pair` (pkg/tests/conftest.py:44-77):

* joint vocabulary: source words ``s{k}``, target words ``t{k}``, and
  3% shared tokens ``x{k}`` spelt identically on both sides (feature 5,
  classifier.py:94-95);
* dictionary: per source word 1 + Poisson(4) translations; the first is
  the true translation tau(s) with p0 ~ U(0.4, 0.9), the rest split
  1 - p0 by a Dirichlet draw; entries below 1e-4 dropped (as
  lexicon.PRUNE_THRESHOLD, lexicon.py:19) and probabilities rounded to
  6 decimals as write_lexicon/read_lexicon round-trip them
  (lexicon.py:153-178);
* sentences: length clip(round(lognormal(3.0, 0.45)), 3, 80), Zipf(1.1)
  word ranks, rendered ``"w1 w2 ... wL."`` (tokenize strips the final
  period, text.py:97-104);
* document pair: N ~ U{40..60}, M = N + U{-5..5}; 60% of source sentences
  have a translation placed monotonically in the target (word -> tau(w)
  w.p. 0.8, another dictionary translation 0.1, a random target word 0.1;
  5% drops and 5% insertions); the other target sentences are unrelated.

Token ids: source word k -> k, target word k -> S + k, shared word
k -> 2S + k.  Dictionary rows exist for ids < S.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .packing import PackedBatch, _ranges

# BASELINE.json configs (index = config number - 1)
CONFIGS = {
    1: dict(n_pairs=1, n_words=1_000, shape=(200, 220)),
    2: dict(n_pairs=10_000, n_words=200_000, shape=None),
    3: dict(n_pairs=1, n_words=200_000, shape=(4096, 4096)),
    4: dict(n_pairs=1_000, n_words=200_000, shape=None),
    5: dict(n_pairs=1_000_000, n_words=200_000, shape=None),
}


def _digits(k: np.ndarray) -> np.ndarray:
    k = np.asarray(k, dtype=np.int64)
    d = np.ones_like(k)
    p = 10
    while p <= max(int(k.max(initial=0)), 1):
        d += k >= p
        p *= 10
    return d


@dataclass
class SynthDictionary:
    n_words: int
    n_shared: int
    tau: np.ndarray  # true translation (target word index) per source word
    src: np.ndarray  # int32 source ids
    tgt: np.ndarray  # int32 target ids (joint space)
    prob: np.ndarray  # float64, 6-decimal values
    row_ptr: np.ndarray = field(default=None)  # CSR over source ids (generation order)

    @property
    def vocab_size(self) -> int:
        return 2 * self.n_words + self.n_shared

    def word(self, token_id: int) -> str:
        s = self.n_words
        if token_id < s:
            return f"s{token_id}"
        if token_id < 2 * s:
            return f"t{token_id - s}"
        return f"x{token_id - 2 * s}"

    def words(self, ids) -> list[str]:
        return [self.word(int(t)) for t in ids]

    def table(self) -> dict[str, dict[str, float]]:
        """dict-of-dicts in the reference Lexicon's shape (lexicon.py:25-26)."""
        table: dict[str, dict[str, float]] = {}
        for s, t, p in zip(self.src.tolist(), self.tgt.tolist(), self.prob.tolist()):
            table.setdefault(self.word(s), {})[self.word(t)] = p
        return table


def make_dictionary(rng: np.random.Generator, n_words: int) -> SynthDictionary:
    s_count = n_words
    n_shared = max(1, (3 * n_words) // 100)
    tau = rng.permutation(s_count)
    k_per = 1 + rng.poisson(4.0, s_count)
    total = int(k_per.sum())
    row = np.repeat(np.arange(s_count), k_per)
    starts = np.concatenate([[0], np.cumsum(k_per)[:-1]])
    first = np.zeros(total, dtype=bool)
    first[starts] = True
    tgt_word = rng.integers(0, s_count, size=total)
    tgt_word[starts] = tau
    p0 = rng.uniform(0.4, 0.9, size=s_count)
    g = rng.gamma(1.0, 1.0, size=total)
    g[starts] = 0.0
    gsum = np.bincount(row, weights=g, minlength=s_count)
    with np.errstate(invalid="ignore", divide="ignore"):
        rest = (1.0 - p0[row]) * g / gsum[row]
    p = np.where(first, p0[row], rest)
    keep = p >= 1e-4
    row, tgt_word, p = row[keep], tgt_word[keep], p[keep]
    # one value per (s, t): a later draw of the same target overwrites the
    # earlier one, as assigning into a dict row does
    key = row.astype(np.int64) * s_count + tgt_word
    _, last_rev = np.unique(key[::-1], return_index=True)
    last = np.sort(len(key) - 1 - last_rev)
    row, tgt_word, p = row[last], tgt_word[last], p[last]
    p6 = np.array([float(f"{v:.6f}") for v in p.tolist()], dtype=np.float64)
    row_ptr = np.zeros(s_count + 1, dtype=np.int64)
    np.cumsum(np.bincount(row, minlength=s_count), out=row_ptr[1:])
    return SynthDictionary(
        n_words=n_words,
        n_shared=n_shared,
        tau=tau,
        src=row.astype(np.int32),
        tgt=(tgt_word + s_count).astype(np.int32),
        prob=p6,
        row_ptr=row_ptr,
    )


@dataclass
class SynthCorpus:
    dictionary: SynthDictionary
    batch: PackedBatch
    # true-translation index pairs: pair p's (i, j) are ref_i/ref_j[ref_off[p]:ref_off[p + 1]]
    ref_off: np.ndarray
    ref_i: np.ndarray
    ref_j: np.ndarray
    _reference: list | None = field(default=None, repr=False)

    @property
    def reference(self) -> list:
        """per pair: list of (i, j) true-translation indices"""
        if self._reference is None:
            ii, jj, off = self.ref_i.tolist(), self.ref_j.tolist(), self.ref_off.tolist()
            self._reference = [list(zip(ii[off[p]: off[p + 1]], jj[off[p]: off[p + 1]])) for p in range(len(off) - 1)]
        return self._reference

    def sentence_text(self, sent: int) -> str:
        b = self.batch
        o = int(b.sent_tok_off[sent])
        ids = b.tokens[o : o + int(b.sent_len[sent])]
        return " ".join(self.dictionary.words(ids)) + "."

    def all_sentences(self) -> list[str]:
        """Every sentence's text (sentence_text for all, vectorised)."""
        return render_sentences(self.batch.tokens, self.batch.sent_len, self.dictionary)

    def pair_sentences(self, pair: int) -> tuple[list[str], list[str]]:
        b = self.batch
        s0, n = int(b.pair_src[pair]), int(b.pair_n[pair])
        t0, m = int(b.pair_tgt[pair]), int(b.pair_m[pair])
        return (
            [self.sentence_text(s0 + i) for i in range(n)],
            [self.sentence_text(t0 + j) for j in range(m)],
        )


def _sentence_lengths(rng, count):
    return np.clip(np.rint(rng.lognormal(3.0, 0.45, size=count)), 3, 80).astype(np.int64)


def _zipf_words(rng, count, n_words):
    return (rng.zipf(1.1, size=count) - 1) % n_words


def _with_shared(rng, ids, d: SynthDictionary):
    mask = rng.random(ids.shape[0]) < 0.03
    shared = 2 * d.n_words + rng.integers(0, d.n_shared, size=ids.shape[0])
    return np.where(mask, shared, ids)


def make_corpus(
    seed: int,
    n_pairs: int,
    n_words: int,
    shape: tuple[int, int] | None = None,
    dictionary: SynthDictionary | None = None,
) -> SynthCorpus:
    """Generate `n_pairs` document pairs (fixed `shape` = (N, M) or the
    C2/C4/C5 distribution)."""
    rng = np.random.default_rng(seed)
    d = dictionary if dictionary is not None else make_dictionary(rng, n_words)
    S = d.n_words
    if shape is None:
        n = rng.integers(40, 61, size=n_pairs)
        m = np.maximum(1, n + rng.integers(-5, 6, size=n_pairs))
    else:
        n = np.full(n_pairs, shape[0], dtype=np.int64)
        m = np.full(n_pairs, shape[1], dtype=np.int64)

    # ---- source sentences (all pairs at once) ----
    ns = int(n.sum())
    src_len = _sentence_lengths(rng, ns)
    src_tok = _with_shared(rng, _zipf_words(rng, int(src_len.sum()), S), d)
    src_off = np.concatenate([[0], np.cumsum(src_len)])
    pair_of_src = np.repeat(np.arange(n_pairs), n)

    # translated source sentences: flag w.p. 0.6, at most M per pair
    flag = rng.random(ns) < 0.6
    csum = np.cumsum(flag) - flag
    first_src = np.concatenate([[0], np.cumsum(n)[:-1]])
    rank_in_pair = csum - (np.cumsum(flag) - flag)[first_src][pair_of_src]
    flag &= rank_in_pair < m[pair_of_src]
    n_tr = np.bincount(pair_of_src, weights=flag, minlength=n_pairs).astype(np.int64)

    # ---- translations of the flagged sentences (token level) ----
    tr_idx = np.flatnonzero(flag)
    tr_len = src_len[tr_idx]
    gather = _ranges(src_off[tr_idx], tr_len)
    w = src_tok[gather]
    is_src_word = w < S
    r = rng.random(w.shape[0])
    rowlen = np.diff(d.row_ptr)
    ws = np.where(is_src_word, w, 0)
    alt = d.tgt[np.minimum(d.row_ptr[ws] + (rng.random(w.shape[0]) * rowlen[ws]).astype(np.int64), len(d.tgt) - 1)]
    rnd = S + d.tau[_zipf_words(rng, w.shape[0], S)]
    mapped = np.where(r < 0.8, S + d.tau[ws], np.where(r < 0.9, alt, rnd))
    mapped = np.where(is_src_word, mapped, w)  # shared tokens stay as they are
    drop = rng.random(w.shape[0]) < 0.05
    ins = rng.random(w.shape[0]) < 0.05
    sent_of_tok = np.repeat(np.arange(tr_idx.size), tr_len)
    keep_cnt = np.bincount(sent_of_tok, weights=~drop, minlength=tr_idx.size)
    # never drop every word of a sentence
    empty = keep_cnt == 0
    if empty.any():
        first_tok = np.concatenate([[0], np.cumsum(tr_len)[:-1]])
        drop[first_tok[empty]] = False
    copies = (~drop).astype(np.int64) + ins
    out_tok = np.repeat(mapped, copies)
    # the second copy of an inserted position becomes a random target word
    out_first = np.concatenate([[0], np.cumsum(copies)[:-1]])
    ins_pos = out_first[ins] + (~drop[ins]).astype(np.int64)
    out_tok[ins_pos] = S + d.tau[_zipf_words(rng, ins_pos.shape[0], S)]
    tr_out_len = np.bincount(sent_of_tok, weights=copies, minlength=tr_idx.size).astype(np.int64)
    tr_out_off = np.concatenate([[0], np.cumsum(tr_out_len)])

    # ---- unrelated target sentences ----
    n_unrel = int((m - n_tr).sum())
    un_len = _sentence_lengths(rng, n_unrel)
    un_tok = _with_shared(rng, S + d.tau[_zipf_words(rng, int(un_len.sum()), S)], d)
    un_off = np.concatenate([[0], np.cumsum(un_len)])

    # ---- assemble: per pair, N source sentences then M target sentences;
    # the pair's translated sentences take the target slots with the k
    # smallest keys (k = its translated count), in slot order
    slot_keys = rng.random(int(m.sum()))
    pair_of_slot = np.repeat(np.arange(n_pairs), m)
    slot_first = np.concatenate([[0], np.cumsum(m)[:-1]])
    order = np.lexsort((slot_keys, pair_of_slot))  # by pair, then key
    rank = np.empty(order.shape[0], dtype=np.int64)
    rank[order] = np.arange(order.shape[0]) - slot_first[pair_of_slot[order]]
    is_tr = rank < n_tr[pair_of_slot]
    # the t-th translated slot of a pair gets the pair's t-th translation,
    # the u-th unrelated slot its u-th unrelated sentence
    tr_before = np.cumsum(is_tr) - is_tr
    un_before = np.cumsum(~is_tr) - (~is_tr)
    # source sentences of the flagged kind, in order, per pair = tr_idx order
    tgt_start = np.where(is_tr, tr_out_off[np.minimum(tr_before, tr_idx.size)],
                         (int(tr_out_off[-1]) + un_off[np.minimum(un_before, n_unrel)]))
    tgt_len = np.where(is_tr, tr_out_len[np.minimum(tr_before, max(tr_idx.size - 1, 0))] if tr_idx.size else 0,
                       un_len[np.minimum(un_before, max(n_unrel - 1, 0))] if n_unrel else 0)
    # sentence order: pair p's N source sentences, then its M target slots
    sent_pair = np.concatenate([np.repeat(np.arange(n_pairs), n), pair_of_slot])
    sent_kind = np.concatenate([np.zeros(ns, dtype=np.int64), np.ones(int(m.sum()), dtype=np.int64)])
    sent_start = np.concatenate([src_off[:-1], int(src_off[-1]) + tgt_start])
    sent_len_all = np.concatenate([src_len, tgt_len])
    sent_order = np.lexsort((sent_kind, sent_pair))  # stable within (pair, kind): source order, slot order
    sent_len = sent_len_all[sent_order]
    pool = np.concatenate([src_tok, out_tok, un_tok])
    tokens = pool[_ranges(sent_start[sent_order], sent_len)]
    pair_src = np.concatenate([[0], np.cumsum(n + m)[:-1]]).astype(np.int64)
    pair_tgt = pair_src + n
    # reference: (local source index of each flagged sentence, its slot)
    ref_cnt = n_tr
    ref_off = np.concatenate([[0], np.cumsum(ref_cnt)]).astype(np.int64)
    ref_i = (tr_idx - first_src[pair_of_src[tr_idx]]).astype(np.int64)
    tr_slots = np.flatnonzero(is_tr)
    ref_j = (tr_slots - slot_first[pair_of_slot[tr_slots]]).astype(np.int64)

    tokens = tokens.astype(np.int32)
    sent_len = sent_len.astype(np.int32)
    batch = PackedBatch.from_token_lengths(
        tokens,
        sent_len,
        sent_chars=_chars(tokens, sent_len, d),
        pair_src=pair_src,
        pair_n=n.astype(np.int32),
        pair_tgt=pair_tgt,
        pair_m=m.astype(np.int32),
    )
    return SynthCorpus(dictionary=d, batch=batch, ref_off=ref_off, ref_i=ref_i, ref_j=ref_j)


def render_sentences(tokens: np.ndarray, sent_len: np.ndarray, d: SynthDictionary) -> list[str]:
    """" ".join(words) + "." per sentence, built as one ASCII buffer."""
    S = d.n_words
    t = np.asarray(tokens, dtype=np.int64)
    prefix = np.where(t < S, ord("s"), np.where(t < 2 * S, ord("t"), ord("x"))).astype(np.uint8)
    num = np.where(t < S, t, np.where(t < 2 * S, t - S, t - 2 * S))
    nd = _digits(num)
    width = 1 + nd + 1  # prefix, digits, then " " or "."
    start = np.zeros(t.shape[0] + 1, dtype=np.int64)
    np.cumsum(width, out=start[1:])
    buf = np.empty(int(start[-1]), dtype=np.uint8)
    buf[start[:-1]] = prefix
    rest = num.copy()
    pos = start[:-1] + nd  # the last digit
    for k in range(int(nd.max(initial=1))):  # digits from the right
        sel = np.flatnonzero(nd > k) if k else slice(None)
        q, r = np.divmod(rest[sel], 10)
        buf[pos[sel] - k] = (ord("0") + r).astype(np.uint8)
        rest[sel] = q
    last = np.zeros(t.shape[0], dtype=bool)
    ends = np.cumsum(sent_len) - 1
    last[ends[sent_len > 0]] = True
    buf[start[1:] - 1] = np.where(last, ord("."), ord(" "))
    text = buf.tobytes().decode("ascii")
    sent_start = start[np.concatenate([[0], np.cumsum(sent_len)[:-1]])].tolist()
    sent_end = start[np.cumsum(sent_len)].tolist()
    return [text[a:b] for a, b in zip(sent_start, sent_end)]


def _chars(tokens: np.ndarray, sent_len: np.ndarray, d: SynthDictionary) -> np.ndarray:
    """len(" ".join(words) + ".") without materialising the strings."""
    S = d.n_words
    t = tokens.astype(np.int64)
    local = np.where(t < S, t, np.where(t < 2 * S, t - S, t - 2 * S))
    word_len = 1 + _digits(local)
    sent_of = np.repeat(np.arange(sent_len.shape[0]), sent_len)
    total = np.bincount(sent_of, weights=word_len, minlength=sent_len.shape[0])
    return (total + sent_len.astype(np.int64)).astype(np.int32)  # (L-1) spaces + "."


def make_config(config: int, seed_base: int = 20261018, n_pairs: int | None = None) -> SynthCorpus:
    spec = CONFIGS[config]
    rng = np.random.default_rng(seed_base + config)
    d = make_dictionary(rng, spec["n_words"])
    return make_corpus(
        seed_base + 1000 + config,
        n_pairs if n_pairs is not None else spec["n_pairs"],
        spec["n_words"],
        spec["shape"],
        dictionary=d,
    )
