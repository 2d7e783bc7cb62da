"""Host side of the boundary: tokenise, map to joint-vocabulary ids, pack.

The reference profiles every sentence inside build_score_matrix
(align.py:112-122 -> classifier.profile_sentence, classifier.py:43-47 ->
tokenize, text.py:97-104) and then compares token *strings*.  Here the
host does exactly that tokenisation once, maps every token string to an
integer in one joint vocabulary shared by both languages and by the
dictionary, and packs the result into the flat arrays of
``bimine_batch`` (include/bimine_b200.h).  Equality of ids is equality
of strings, so the device computes the same set memberships.
"""

from __future__ import annotations

import dataclasses
from dataclasses import dataclass
from typing import Iterable, Sequence

import numpy as np

from .text import tokenize


class Vocabulary:
    """str -> int32 id, grown on demand; one instance per Lexicon (Python dict)."""

    __slots__ = ("ids", "words")
    native = False

    def __init__(self) -> None:
        self.ids: dict[str, int] = {}
        self.words: list[str] = []

    def __len__(self) -> int:
        return len(self.words)

    def get(self, word: str) -> int:
        i = self.ids.get(word)
        if i is None:
            i = len(self.words)
            self.ids[word] = i
            self.words.append(word)
        return i

    def add_many(self, words) -> np.ndarray:
        return np.fromiter((self.get(w) for w in words), dtype=np.int32)


def _token_buffer(n: int) -> np.ndarray:
    """int32 output of the tokenizer: page-locked when a GPU is present
    (torch's caching host allocator: the block is reused call after call
    instead of faulting in and unmapping ~10^8 fresh bytes, and the batch
    then uploads without staging), else plain memory."""
    if n >= (1 << 20):
        try:
            import torch

            if torch.cuda.is_available():
                return torch.empty(4 * n, dtype=torch.uint8, pin_memory=True).numpy().view(np.int32)
        except Exception:  # pragma: no cover - no usable CUDA runtime
            pass
    return np.empty(n, dtype=np.int32)


def _pyhost():
    """The CPython helper module (csrc/pyhost.c), built with the library."""
    from . import _pyhost as m

    return m


def _utf8_offsets(strings: list[str]) -> tuple[bytes, np.ndarray]:
    """The strings' UTF-8 bytes back to back, and their byte offsets."""
    off = np.zeros(len(strings) + 1, dtype=np.int64)
    if all(map(str.isascii, strings)):  # (O(1) per string) byte offsets = character offsets
        np.cumsum(np.fromiter(map(len, strings), dtype=np.int64, count=len(strings)), out=off[1:])
        return "".join(strings).encode("ascii"), off
    enc = [x.encode("utf-8", "surrogatepass") for x in strings]
    np.cumsum(np.fromiter(map(len, enc), dtype=np.int64, count=len(enc)), out=off[1:])
    return b"".join(enc), off


class NativeVocabulary:
    """The same mapping kept in libbimine_b200.so (bimine_vocab_*), with the
    native tokenizer (bimine_tokenize_batch) for ASCII and Latin-1 /
    Latin Extended-A sentences (the Python rules for the rest)."""

    native = True

    def __init__(self) -> None:
        import ctypes

        from . import _native as N

        self._N = N
        self._L = N.load(require_gpu=False)
        h = ctypes.c_void_p()
        N.check(self._L.bimine_vocab_create(ctypes.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                self._L.bimine_vocab_destroy(h)
            except Exception:
                pass

    def __len__(self) -> int:
        return int(self._L.bimine_vocab_size(self._h))

    def add_many(self, words) -> np.ndarray:
        words = list(words)
        data, off = _utf8_offsets(words)
        ids = np.empty(max(len(words), 1), dtype=np.int32)
        N = self._N
        N.check(self._L.bimine_vocab_add_batch(self._h, data, N.ptr(off, N._i64p), len(words), N.ptr(ids, N._i32p)))
        return ids[: len(words)]

    def get(self, word: str) -> int:
        return int(self.add_many([word])[0])

    def _in_place(self, n: int, ptrs, blen, prefix):
        """bimine_tokenize_ptrs over n sentences' own storage."""
        N = self._N
        lens = np.empty(max(n, 1), dtype=np.int32)
        uniq = np.empty(max(n, 1), dtype=np.int32)
        chars = np.empty(max(n, 1), dtype=np.int32)
        nt = np.zeros(1, dtype=np.int64)
        # first try room for one token per 5 characters (natural text has
        # 5-7); denser text is refused with the vocabulary unchanged and
        # tokenised again with the worst-case bound
        for cap in (int(prefix[n]) // 5 + n + 1, int(prefix[n]) // 2 + n + 1):
            tokens = _token_buffer(cap)
            rc = self._L.bimine_tokenize_ptrs(self._h, ptrs.ctypes.data, N.ptr(blen, N._i64p), n,
                                              N.ptr(prefix, N._i64p), N.ptr(tokens, N._i32p), cap, N.ptr(nt, N._i64p),
                                              N.ptr(lens, N._i32p), N.ptr(uniq, N._i32p), N.ptr(chars, N._i32p))
            if rc != N.BIMINE_E_LIMIT:
                break
        N.check(rc)
        return tokens[: int(nt[0])], lens[:n], uniq[:n], chars[:n]

    def tokenize_docs(self, docs, n: int, start: np.ndarray):
        """tokenize() of the n sentences of `docs`, a list of (source
        sentences, target sentences), pair by pair, source first (pair d's
        first sentence is start[d], start[-1] == n) -- read in
        place, without a flat list; None unless every pair is a tuple or
        list of two tuples or lists of compact ASCII str (the caller then
        flattens them for tokenize())."""
        ptrs, blen, prefix = (np.empty(max(n, 1), dtype=np.int64), np.empty(max(n, 1), dtype=np.int64),
                              np.empty(n + 1, dtype=np.int64))
        if not (n and type(docs) is list and _pyhost().docs_view(docs, ptrs, blen, prefix, start)):
            return None
        return self._in_place(n, ptrs, blen, prefix)

    def tokenize(self, sentences: list[str]):
        """(tokens int32, len, uniq, chars) per sentence with the reference's
        tokenize(); a sentence with no token has len 0.  ASCII sentences are
        read in place (their str storage); others go through one UTF-8
        buffer."""
        N = self._N
        n = len(sentences)
        ptrs, blen, prefix = (np.empty(max(n, 1), dtype=np.int64), np.empty(max(n, 1), dtype=np.int64),
                              np.empty(n + 1, dtype=np.int64))
        if n and type(sentences) is list and _pyhost().str_view(sentences, ptrs, blen, prefix):
            return self._in_place(n, ptrs, blen, prefix)  # every sentence a compact ASCII str
        lens = np.empty(max(n, 1), dtype=np.int32)
        uniq = np.empty(max(n, 1), dtype=np.int32)
        chars = np.empty(max(n, 1), dtype=np.int32)
        nt = np.zeros(1, dtype=np.int64)
        data, off = _utf8_offsets(sentences)
        cap = len(data) // 2 + n + 1
        tokens = np.empty(cap, dtype=np.int32)
        N.check(self._L.bimine_tokenize_batch(self._h, data, N.ptr(off, N._i64p), n, N.ptr(tokens, N._i32p), cap,
                                              N.ptr(nt, N._i64p), N.ptr(lens, N._i32p), N.ptr(uniq, N._i32p),
                                              N.ptr(chars, N._i32p)))
        tokens, lens, uniq, chars = tokens[: int(nt[0])], lens[:n], uniq[:n], chars[:n]
        slow = np.flatnonzero(lens < 0)
        if slow.size:  # code points >= U+0180 (or U+0130): Python's Unicode rules, same vocabulary
            starts = np.zeros(n + 1, dtype=np.int64)
            np.cumsum(np.maximum(lens, 0), out=starts[1:])
            pieces = []
            for k in range(n):
                if lens[k] >= 0:
                    pieces.append(tokens[starts[k] : starts[k] + lens[k]])
                else:
                    ids = self.add_many(tokenize(sentences[k]))
                    pieces.append(ids)
                    lens[k] = ids.shape[0]
                    uniq[k] = len(set(ids.tolist()))
                    chars[k] = len(sentences[k])
            tokens = np.concatenate(pieces) if pieces else np.zeros(0, np.int32)
        return tokens.astype(np.int32, copy=False), lens, uniq, chars


def new_vocabulary():
    """The native vocabulary when libbimine_b200.so is built, else the dict one."""
    try:
        return NativeVocabulary()
    except Exception:
        return Vocabulary()


@dataclass
class PackedBatch:
    tokens: np.ndarray  # int32 [T]; with token_bytes == 3: uint8 [3 T], 24-bit little-endian ids
    sent_tok_off: np.ndarray  # int64 [S]
    sent_len: np.ndarray  # int32 [S]
    sent_uniq: np.ndarray  # int32 [S]
    sent_chars: np.ndarray  # int32 [S]
    pair_src: np.ndarray  # int64 [P]
    pair_n: np.ndarray  # int32 [P]
    pair_tgt: np.ndarray  # int64 [P]
    pair_m: np.ndarray  # int32 [P]
    pair_sim_off: np.ndarray  # int64 [P]
    token_bytes: int = 4  # 3: the compact wire form of the ids (with_24bit_tokens)
    sent_bytes: int = 4  # 2: sent_len / sent_uniq / sent_chars as uint16 (with_narrow_sentences)

    @property
    def n_pairs(self) -> int:
        return int(self.pair_n.shape[0])

    def with_24bit_tokens(self) -> "PackedBatch":
        """The same batch with its token ids packed in 3 bytes each (every id
        in [0, 2^24)): the form bimine_mine_host uploads a quarter faster.
        The kernels read it directly; host-side consumers want int32."""
        if self.token_bytes == 3:
            return self
        t = np.ascontiguousarray(self.tokens, dtype=np.int32)
        if t.size and (int(t.min()) < 0 or int(t.max()) >= 1 << 24):
            raise ValueError("token ids outside [0, 2^24) need the int32 form")
        packed = np.ascontiguousarray(t.view(np.uint8).reshape(-1, 4)[:, :3]).reshape(-1)
        return dataclasses.replace(self, tokens=packed, token_bytes=3)

    def with_narrow_sentences(self) -> "PackedBatch":
        """The same batch with sent_len, sent_uniq and sent_chars as uint16
        (every value below 2^16; otherwise the batch is returned as is):
        the form whose sentence arrays bimine_mine_host uploads in half the
        time.  For bimine_mine_host only; other consumers want int32."""
        if self.sent_bytes == 2:
            return self
        arrs = (self.sent_len, self.sent_uniq, self.sent_chars)
        if any(a.size and (int(a.min()) < 0 or int(a.max()) >= 1 << 16) for a in arrs):
            return self
        narrow = [np.ascontiguousarray(a, dtype=np.uint16) for a in arrs]
        return dataclasses.replace(self, sent_len=narrow[0], sent_uniq=narrow[1], sent_chars=narrow[2], sent_bytes=2)

    def int32_tokens(self) -> np.ndarray:
        """The ids as int32 whatever the stored form."""
        if self.token_bytes != 3:
            return self.tokens
        b = self.tokens.reshape(-1, 3).astype(np.int32)
        return b[:, 0] | (b[:, 1] << 8) | (b[:, 2] << 16)

    @property
    def n_sentences(self) -> int:
        return int(self.sent_len.shape[0])

    @property
    def n_tokens(self) -> int:
        return int(self.tokens.shape[0]) // (3 if self.token_bytes == 3 else 1)

    @property
    def n_cells(self) -> int:
        return int(self.pair_sim_off[-1] + int(self.pair_n[-1]) * int(self.pair_m[-1])) if self.n_pairs else 0

    def match_capacity(self) -> np.ndarray:
        """Per-pair slot offsets for matches (capacity min(N, M) each) and total."""
        cap = np.minimum(self.pair_n, self.pair_m).astype(np.int64)
        off = np.zeros(self.n_pairs + 1, dtype=np.int64)
        np.cumsum(cap, out=off[1:])
        return off

    def nbytes(self) -> int:
        return sum(
            a.nbytes
            for a in (
                self.tokens, self.sent_tok_off, self.sent_len, self.sent_uniq,
                self.sent_chars, self.pair_src, self.pair_n, self.pair_tgt,
                self.pair_m, self.pair_sim_off,
            )
        )

    @staticmethod
    def from_token_lengths(
        tokens: np.ndarray,
        sent_len: np.ndarray,
        sent_chars: np.ndarray,
        pair_src: np.ndarray,
        pair_n: np.ndarray,
        pair_tgt: np.ndarray,
        pair_m: np.ndarray,
        sent_uniq: np.ndarray | None = None,
    ) -> "PackedBatch":
        tokens = np.ascontiguousarray(tokens, dtype=np.int32)
        sent_len = np.ascontiguousarray(sent_len, dtype=np.int32)
        off = np.zeros(sent_len.shape[0], dtype=np.int64)
        if sent_len.shape[0] > 1:
            np.cumsum(sent_len[:-1], out=off[1:])
        if sent_uniq is None:
            sent_uniq = unique_counts(tokens, sent_len)
        pair_n = np.ascontiguousarray(pair_n, dtype=np.int32)
        pair_m = np.ascontiguousarray(pair_m, dtype=np.int32)
        cells = pair_n.astype(np.int64) * pair_m.astype(np.int64)
        sim_off = np.zeros(pair_n.shape[0], dtype=np.int64)
        if pair_n.shape[0] > 1:
            np.cumsum(cells[:-1], out=sim_off[1:])
        return PackedBatch(
            tokens=tokens,
            sent_tok_off=off,
            sent_len=sent_len,
            sent_uniq=np.ascontiguousarray(sent_uniq, dtype=np.int32),
            sent_chars=np.ascontiguousarray(sent_chars, dtype=np.int32),
            pair_src=np.ascontiguousarray(pair_src, dtype=np.int64),
            pair_n=pair_n,
            pair_tgt=np.ascontiguousarray(pair_tgt, dtype=np.int64),
            pair_m=pair_m,
            pair_sim_off=sim_off,
        )

    def select(self, pairs: Sequence[int] | np.ndarray) -> "PackedBatch":
        """Sub-batch of the given pairs (order kept), re-packed contiguously."""
        pairs = np.asarray(pairs, dtype=np.int64)
        pn = self.pair_n[pairs].astype(np.int64)
        pm = self.pair_m[pairs].astype(np.int64)
        # per pair: its source sentences, then its target sentences
        sent_idx = _ranges(np.stack([self.pair_src[pairs], self.pair_tgt[pairs]], axis=1).ravel(),
                           np.stack([pn, pm], axis=1).ravel())
        lens = self.sent_len[sent_idx]
        tok_idx = _ranges(self.sent_tok_off[sent_idx], lens)
        starts = np.zeros(pairs.shape[0], dtype=np.int64)
        if pairs.shape[0] > 1:
            np.cumsum((pn + pm)[:-1], out=starts[1:])
        return PackedBatch.from_token_lengths(
            self.tokens[tok_idx], lens, self.sent_chars[sent_idx],
            starts, pn, starts + pn, pm, sent_uniq=self.sent_uniq[sent_idx],
        )


def _ranges(starts, lens) -> np.ndarray:
    """concatenate(arange(s, s + l) for s, l in zip(starts, lens)), vectorised."""
    lens = np.asarray(lens, dtype=np.int64)
    total = int(lens.sum())
    if total == 0:
        return np.zeros(0, dtype=np.int64)
    first = np.zeros(lens.shape[0], dtype=np.int64)
    np.cumsum(lens[:-1], out=first[1:])
    return np.repeat(np.asarray(starts, dtype=np.int64) - first, lens) + np.arange(total, dtype=np.int64)


def unique_counts(tokens: np.ndarray, sent_len: np.ndarray) -> np.ndarray:
    """len(set(tokens)) per sentence, vectorised."""
    n_sent = sent_len.shape[0]
    if tokens.shape[0] == 0:
        return np.zeros(n_sent, dtype=np.int32)
    sent_of = np.repeat(np.arange(n_sent, dtype=np.int64), sent_len)
    key = sent_of << 32 | tokens.astype(np.int64) & 0xFFFFFFFF
    key.sort()
    first = np.ones(key.shape[0], dtype=bool)
    first[1:] = key[1:] != key[:-1]
    return np.bincount(key[first] >> 32, minlength=n_sent).astype(np.int32)


class SentenceError(ValueError):
    """An untokenizable sentence, with the side/index prefix the reference
    adds in build_score_matrix (align.py:112-119)."""


def profile_ids(sentence: str, vocab: Vocabulary) -> list[int]:
    """profile_sentence (classifier.py:43-47) down to token ids."""
    tokens = tokenize(sentence)
    if not tokens:
        raise ValueError(f"untokenizable sentence: {sentence!r}")
    get = vocab.get
    return [get(t) for t in tokens]


@dataclass
class PackedDocuments:
    """Result of pack_documents: the batch of the pairs that tokenise, and
    the bookkeeping to map matches back to sentence text."""

    batch: PackedBatch | None  # None when no pair tokenises
    docs: list  # the input pairs: (source sentences, target sentences)
    start: np.ndarray  # [P + 1] first sentence of input pair k, counting source then target sentences pair by pair
    n_src: np.ndarray  # [P] source sentence count per input pair
    ok: np.ndarray  # [P] bool: input pair k is in the batch
    errors: dict  # input pair -> the reference's ValueError message


def pack_documents(vocab, pairs) -> PackedDocuments:
    """Tokenise and pack many (source_sentences, target_sentences) at once
    (one native tokenizer call over the sentences' own storage; a pair whose
    sentence does not tokenise is left out with the message the reference
    raises for it, align.py:109-119)."""
    import itertools

    pairs = pairs if type(pairs) is list else list(pairs)
    P = len(pairs)
    ns = np.fromiter((len(x[0]) for x in pairs), dtype=np.int64, count=P)
    nt = np.fromiter((len(x[1]) for x in pairs), dtype=np.int64, count=P)
    start = np.zeros(P + 1, dtype=np.int64)
    np.cumsum(ns + nt, out=start[1:])
    S = int(start[P])
    res = vocab.tokenize_docs(pairs, S, start) if getattr(vocab, "native", False) else None
    if res is not None:
        tokens, lens, uniq, chars = res
    else:
        flat = list(itertools.chain.from_iterable(itertools.chain(x[0], x[1]) for x in pairs))
        if getattr(vocab, "native", False):
            tokens, lens, uniq, chars = vocab.tokenize(flat)
        else:  # the dict vocabulary: the Python rules sentence by sentence
            ids = []
            for sent in flat:
                ids.append(np.asarray([vocab.get(t) for t in tokenize(sent)], dtype=np.int32))
            lens = np.fromiter(map(len, ids), dtype=np.int32, count=len(ids))
            uniq = np.fromiter((len(set(x.tolist())) for x in ids), dtype=np.int32, count=len(ids))
            chars = np.fromiter(map(len, flat), dtype=np.int32, count=len(flat))
            tokens = np.concatenate(ids) if ids else np.zeros(0, np.int32)
    lens = lens[:S]
    zero = np.zeros(S + 1, dtype=np.int64)
    np.cumsum(lens == 0, out=zero[1:])
    ok = (ns > 0) & (nt > 0) & (zero[start[1:]] == zero[start[:-1]])
    errors = {}
    for k in np.flatnonzero(~ok).tolist():  # the reference's messages
        if not ns[k] or not nt[k]:
            errors[k] = "both sentence sequences must be non-empty"
            continue
        bad = int(np.flatnonzero(lens[start[k]: start[k + 1]] == 0)[0])
        side, index = ("source", bad) if bad < ns[k] else ("target", bad - int(ns[k]))
        text = pairs[k][0 if side == "source" else 1][index]
        errors[k] = f"{side} sentence {index}: untokenizable sentence: {text!r}"
    keep = np.flatnonzero(ok)
    batch = None
    if keep.size:
        if keep.size == P:
            tok, sl, su, sc = tokens, lens, uniq[:S], chars[:S]
            first = start[:-1]
        else:
            sent_keep = np.repeat(ok, ns + nt)
            tok = tokens[np.repeat(sent_keep, lens)]
            sl, su, sc = lens[sent_keep], uniq[:S][sent_keep], chars[:S][sent_keep]
            first = np.zeros(keep.size, dtype=np.int64)
            np.cumsum((ns + nt)[keep][:-1], out=first[1:])
        batch = PackedBatch.from_token_lengths(tok, sl, sc, first, ns[keep], first + ns[keep], nt[keep],
                                               sent_uniq=su)
    return PackedDocuments(batch=batch, docs=pairs, start=start, n_src=ns, ok=ok, errors=errors)


class BatchBuilder:
    """Accumulates document pairs (as sentence strings) into a PackedBatch."""

    def __init__(self, vocab) -> None:
        self.vocab = vocab
        self.parts: list[PackedBatch] = []
        self.n_pairs = 0

    def _profiles(self, sentences: Sequence[str], side: str) -> list[list[int]]:
        out = []
        for index, sentence in enumerate(sentences):
            try:
                out.append(profile_ids(sentence, self.vocab))
            except ValueError as exc:
                raise SentenceError(f"{side} sentence {index}: {exc}") from None
        return out

    def add_pair(self, source: Sequence[str], target: Sequence[str]) -> int:
        """Tokenise and append one pair; raises ValueError with the
        reference's messages (align.py:109-119) and leaves the builder
        unchanged on error.  Returns the pair's index in the batch."""
        [res] = self.add_pairs([(source, target)])
        if isinstance(res, str):
            raise ValueError(res)
        return res

    def add_pairs(self, pairs) -> list:
        """Append many (source_sentences, target_sentences) at once.  Returns,
        per input pair, its batch index or the ValueError message the
        reference would raise for it (the pair is then not appended)."""
        if not pairs:
            return []
        pd = pack_documents(self.vocab, pairs)
        out: list = [None] * len(pairs)
        for k, msg in pd.errors.items():
            out[k] = msg
        for b, k in enumerate(np.flatnonzero(pd.ok).tolist()):
            out[k] = self.n_pairs + b
        if pd.batch is not None:
            self.parts.append(pd.batch)
            self.n_pairs += pd.batch.n_pairs
        return out

    def build(self) -> PackedBatch:
        if len(self.parts) == 1:
            return self.parts[0]
        if not self.parts:
            z32, z64 = np.zeros(0, np.int32), np.zeros(0, np.int64)
            return PackedBatch(z32, z64, z32, z32, z32, z64, z32, z64, z32, z64)
        s_base = np.cumsum([0] + [p.n_sentences for p in self.parts[:-1]])
        return PackedBatch.from_token_lengths(
            np.concatenate([p.tokens for p in self.parts]),
            np.concatenate([p.sent_len for p in self.parts]),
            np.concatenate([p.sent_chars for p in self.parts]),
            np.concatenate([p.pair_src + b for p, b in zip(self.parts, s_base)]),
            np.concatenate([p.pair_n for p in self.parts]),
            np.concatenate([p.pair_tgt + b for p, b in zip(self.parts, s_base)]),
            np.concatenate([p.pair_m for p in self.parts]),
            sent_uniq=np.concatenate([p.sent_uniq for p in self.parts]),
        )


def lexicon_arrays(entries: Iterable[tuple[str, str, float]], vocab):
    """COO (src, tgt, prob) arrays of a lexicon in its iteration order."""
    ss, ts, ps = [], [], []
    for s, t, p in entries:
        ss.append(s)
        ts.append(t)
        ps.append(float(p))
    words = [w for pair in zip(ss, ts) for w in pair]
    ids = vocab.add_many(words) if words else np.zeros(0, np.int32)
    return (
        np.ascontiguousarray(ids[0::2], dtype=np.int32),
        np.ascontiguousarray(ids[1::2], dtype=np.int32),
        np.asarray(ps, dtype=np.float64),
    )
