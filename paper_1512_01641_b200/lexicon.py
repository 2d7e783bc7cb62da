"""Bilingual dictionary (reference lexicon.py:22-59, 153-178) and its EM
estimation from sentence pairs (``build_lexicon``, lexicon.py:60-120; the
rounds run on the GPU, csrc/lexicon_em.cuh).

``Lexicon`` keeps the reference's read API (dict of dicts).  Its device
form -- a CSR over joint-vocabulary source ids, replicated per GPU --
is built lazily by ``align`` through the C ABI (bimine_dict_create) and
cached per (lexicon, device).  Any object with ``items()`` yielding
(source, target, p) -- including the reference's own Lexicon -- is
accepted by the mining API.
"""

from __future__ import annotations

import os
from collections import defaultdict
from typing import Iterator, Mapping, Sequence

import numpy as np

# Entries below this probability are dropped after the final round (lexicon.py:18-19).
PRUNE_THRESHOLD = 1e-4


class Lexicon:
    """Immutable token translation table with per-source probabilities."""

    def __init__(self, table: Mapping[str, Mapping[str, float]]):
        self._table = {s: dict(row) for s, row in table.items()}

    def prob(self, source_token: str, target_token: str) -> float:
        return self._table.get(source_token, {}).get(target_token, 0.0)

    def translations(self, source_token: str) -> Mapping[str, float]:
        return self._table.get(source_token, {})

    def source_tokens(self) -> Iterator[str]:
        return iter(self._table)

    def items(self) -> Iterator[tuple[str, str, float]]:
        for s, row in self._table.items():
            for t, p in row.items():
                yield s, t, p

    def __len__(self) -> int:
        return sum(len(row) for row in self._table.values())

    def __eq__(self, other: object) -> bool:
        return isinstance(other, Lexicon) and self._table == other._table

    __hash__ = object.__hash__


def write_lexicon(lexicon, path: str | os.PathLike) -> None:
    """``source<TAB>target<TAB>p`` rows, sorted by source, descending p, target."""
    entries = sorted(lexicon.items(), key=lambda e: (e[0], -e[2], e[1]))
    with open(path, "w", encoding="utf-8") as handle:
        for s, t, p in entries:
            handle.write(f"{s}\t{t}\t{p:.6f}\n")


def read_lexicon(path: str | os.PathLike) -> Lexicon:
    """TSV reader; a repeated (source, target) keeps the last value."""
    table: dict[str, dict[str, float]] = defaultdict(dict)
    with open(path, encoding="utf-8") as handle:
        for lineno, line in enumerate(handle, 1):
            line = line.rstrip("\n")
            if not line:
                continue
            fields = line.split("\t")
            if len(fields) != 3:
                raise ValueError(
                    f"{path}: line {lineno}: expected 3 tab-separated fields, got {len(fields)}"
                )
            table[fields[0]][fields[1]] = float(fields[2])
    return Lexicon(table)


def build_lexicon(parallel: Sequence[tuple[str, str]], iterations: int,
                  prune_threshold: float = PRUNE_THRESHOLD) -> Lexicon:
    """EM estimate of p(t | s) from sentence pairs, bit-identical to the
    reference's float64 arithmetic (lexicon.py:60-120).

    Host: tokenise (pairs with an empty side are skipped), give source and
    target tokens integer ids, build every source token's support (all
    co-occurring targets, uniform start 1 / |support|) and the corpus-order
    occurrence list of every source id.  Device: ``iterations`` EM rounds
    (bimine_lexicon_em).  Host: drop entries below ``prune_threshold``
    and empty rows.
    """
    from . import _native as N
    from .text import tokenize

    if not parallel:
        raise ValueError("no training pairs")
    if iterations < 1:
        raise ValueError("iterations must be >= 1")
    src_ids: dict[str, int] = {}
    tgt_ids: dict[str, int] = {}
    pairs_s, pairs_t = [], []
    for source_sentence, target_sentence in parallel:
        st, tt = tokenize(source_sentence), tokenize(target_sentence)
        if st and tt:
            pairs_s.append(np.fromiter((src_ids.setdefault(w, len(src_ids)) for w in st), np.int64, len(st)))
            pairs_t.append(np.fromiter((tgt_ids.setdefault(w, len(tgt_ids)) for w in tt), np.int64, len(tt)))
    if not pairs_s:
        raise ValueError("no training pairs")
    n_src, n_tgt, P = len(src_ids), len(tgt_ids), len(pairs_s)
    # support: unique (s, t) co-occurrences, sorted by s then t
    keys = np.unique(np.concatenate([(np.unique(a)[:, None] * n_tgt + np.unique(b)[None, :]).ravel()
                                     for a, b in zip(pairs_s, pairs_t)]))
    row_s = keys // n_tgt
    row_tgt = (keys % n_tgt).astype(np.int32)
    row_len = np.bincount(row_s, minlength=n_src)
    row_ptr = np.zeros(n_src + 1, dtype=np.int64)
    np.cumsum(row_len, out=row_ptr[1:])
    prob = 1.0 / row_len[row_s].astype(np.float64)  # lexicon.py:92-94, one IEEE division per row
    # occurrences of every source id in corpus order (stable sort keeps it)
    occ_s = np.concatenate(pairs_s)
    occ_p = np.repeat(np.arange(P, dtype=np.int32), [a.size for a in pairs_s])
    perm = np.argsort(occ_s, kind="stable")
    occ_pair = occ_p[perm]
    occ_ptr = np.zeros(n_src + 1, dtype=np.int64)
    np.cumsum(np.bincount(occ_s, minlength=n_src), out=occ_ptr[1:])
    tgt_off = np.zeros(P + 1, dtype=np.int32)
    np.cumsum([b.size for b in pairs_t], out=tgt_off[1:])
    tgt_tok = np.concatenate(pairs_t).astype(np.int32)

    import torch

    L = N.load()
    dev = torch.device("cuda", torch.cuda.current_device())
    t = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for k, v in
         dict(tgt_off=tgt_off, tgt_tok=tgt_tok, row_ptr=row_ptr, row_tgt=row_tgt, prob=prob,
              alive=np.ones(prob.size, dtype=np.uint8), occ_ptr=occ_ptr, occ_pair=occ_pair).items()}
    N.check(L.bimine_lexicon_em(t["tgt_off"].data_ptr(), t["tgt_tok"].data_ptr(), P, n_src, t["row_ptr"].data_ptr(),
                                t["row_tgt"].data_ptr(), int(prob.size), t["prob"].data_ptr(), t["alive"].data_ptr(),
                                t["occ_ptr"].data_ptr(), t["occ_pair"].data_ptr(), int(iterations),
                                torch.cuda.current_stream().cuda_stream))
    prob = t["prob"].cpu().numpy()
    alive = t["alive"].cpu().numpy().astype(bool)
    keep = alive & (prob >= prune_threshold) if prune_threshold > 0.0 else alive
    src_words = np.array(list(src_ids), dtype=object)
    tgt_words = np.array(list(tgt_ids), dtype=object)
    table: dict[str, dict[str, float]] = {}
    for sw, tw, p in zip(src_words[row_s[keep]], tgt_words[row_tgt[keep]], prob[keep]):
        table.setdefault(sw, {})[tw] = float(p)
    return Lexicon(table)


def merge_title_lexicon(lexicon, titles) -> tuple["Lexicon", int]:
    """Fold single-token title pairs into the lexicon (lexicon.py:128-150):
    p = max(existing, 0.5), the source row renormalised by Python's sum();
    titles that are not one token on each side are skipped and counted."""
    from .text import tokenize

    table = {s: dict(lexicon.translations(s)) for s in lexicon.source_tokens()}
    skipped = 0
    for source_title, target_title in titles:
        st, tt = tokenize(source_title), tokenize(target_title)
        if len(st) != 1 or len(tt) != 1:
            skipped += 1
            continue
        row = table.setdefault(st[0], {})
        row[tt[0]] = max(row.get(tt[0], 0.0), 0.5)
        total = sum(row.values())
        table[st[0]] = {t: p / total for t, p in row.items()}
    return Lexicon(table), skipped
