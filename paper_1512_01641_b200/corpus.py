"""Document-pair inputs of the mining API and the corpus files around it.

Value types: reference corpus.py:21-51.  File-level drop-in for
``bimine mine``: the paired-corpus directory
(``pairs.tsv`` + ``sentences.tsv``, corpus.py:225-301), the mined bitext
(``%.4f\tsource\ttarget``, corpus.py:203-222) and the field escaping of
titles and topic ids (corpus.py:68-80).  Functions in ``align`` accept any
object with the same attributes (duck typing), so the reference's own
``bimine.corpus.DocumentPair`` instances work too.
"""

from __future__ import annotations

import os
import re
from dataclasses import dataclass
from typing import Iterable, Sequence


@dataclass(frozen=True)
class Document:
    """One cleaned, segmented article in one language."""

    id: str
    lang: str
    title: str
    sentences: tuple[str, ...]

    def __post_init__(self) -> None:
        if not self.id:
            raise ValueError("document id must be non-empty")
        if not self.sentences:
            raise ValueError(f"document {self.id} has no sentences")
        if any(not s.strip() for s in self.sentences):
            raise ValueError(f"document {self.id} contains an empty sentence")


@dataclass(frozen=True)
class DocumentPair:
    """Two topic-aligned articles in different languages."""

    topic_id: str
    source: Document
    target: Document

    def __post_init__(self) -> None:
        if self.source.lang == self.target.lang:
            raise ValueError(
                f"pair {self.topic_id}: both sides have language {self.source.lang!r}"
            )


# ---- field escaping (corpus.py:68-80): backslash, tab and newline
_ESCAPE_TABLE = str.maketrans({"\\": "\\\\", "\t": "\\t", "\n": "\\n"})
_UNESCAPE = re.compile(r"\\([\\tn])")
_UNESCAPED = {"\\": "\\", "t": "\t", "n": "\n"}


def escape_field(text: str) -> str:
    return text.translate(_ESCAPE_TABLE)


def unescape_field(text: str) -> str:
    return _UNESCAPE.sub(lambda m: _UNESCAPED[m.group(1)], text)


# ---- mined bitext (corpus.py:203-222)
def write_bitext(path: str | os.PathLike, rows: Iterable[tuple[float, str, str]]) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        fh.writelines(f"{float(score):.4f}\t{src}\t{tgt}\n" for score, src, tgt in rows)


def read_bitext(path: str | os.PathLike) -> list[tuple[float, str, str]]:
    out = []
    with open(path, encoding="utf-8") as fh:
        for lineno, raw in enumerate(fh, 1):
            line = raw.rstrip("\n")
            if not line:
                continue
            fields = line.split("\t")
            if len(fields) != 3:
                raise ValueError(f"{path}: line {lineno}: expected 3 tab-separated fields, got {len(fields)}")
            out.append((float(fields[0]), fields[1], fields[2]))
    return out


# ---- paired corpus directory (corpus.py:225-301)
PAIRS_FILE = "pairs.tsv"
SENTENCES_FILE = "sentences.tsv"


def save_corpus(pairs: Sequence[DocumentPair], out_dir: str | os.PathLike) -> None:
    """pairs.tsv: topic, then id / lang / title of each side; sentences.tsv:
    topic, side (src|tgt), index, sentence -- one row per sentence."""
    os.makedirs(out_dir, exist_ok=True)
    with open(os.path.join(out_dir, PAIRS_FILE), "w", encoding="utf-8") as fh:
        for pr in pairs:
            cols = [escape_field(pr.topic_id)]
            for doc in (pr.source, pr.target):
                cols += [doc.id, doc.lang, escape_field(doc.title)]
            fh.write("\t".join(cols) + "\n")
    with open(os.path.join(out_dir, SENTENCES_FILE), "w", encoding="utf-8") as fh:
        for pr in pairs:
            topic = escape_field(pr.topic_id)
            for side, doc in (("src", pr.source), ("tgt", pr.target)):
                fh.writelines(f"{topic}\t{side}\t{k}\t{sent}\n" for k, sent in enumerate(doc.sentences))


def _rows(path):
    with open(path, encoding="utf-8") as fh:
        for lineno, raw in enumerate(fh, 1):
            line = raw.rstrip("\n")
            if line:
                yield lineno, line.split("\t")


def load_corpus(corpus_dir: str | os.PathLike) -> list[DocumentPair]:
    """Read a paired-corpus directory; each side's sentences are ordered by
    their index (sentences of a topic/side may appear in any order)."""
    pairs_path = os.path.join(corpus_dir, PAIRS_FILE)
    sentences_path = os.path.join(corpus_dir, SENTENCES_FILE)
    by_doc: dict[tuple[str, str], list[tuple[int, str]]] = {}
    for lineno, f in _rows(sentences_path):
        if len(f) != 4:
            raise ValueError(f"{sentences_path}: line {lineno}: malformed sentence row")
        by_doc.setdefault((unescape_field(f[0]), f[1]), []).append((int(f[2]), f[3]))

    def sentences_of(topic: str, side: str) -> tuple[str, ...]:
        return tuple(text for _, text in sorted(by_doc.get((topic, side), [])))

    out: list[DocumentPair] = []
    for lineno, f in _rows(pairs_path):
        if len(f) != 7:
            raise ValueError(f"{pairs_path}: line {lineno}: malformed pair row")
        topic = unescape_field(f[0])
        src = Document(id=f[1], lang=f[2], title=unescape_field(f[3]), sentences=sentences_of(topic, "src"))
        tgt = Document(id=f[4], lang=f[5], title=unescape_field(f[6]), sentences=sentences_of(topic, "tgt"))
        out.append(DocumentPair(topic_id=topic, source=src, target=tgt))
    return out


# ---- two-column files: training pairs, title / document links (corpus.py:170-200)
def _two_fields(path) -> list[tuple[str, str]]:
    out = []
    with open(path, encoding="utf-8") as fh:
        for lineno, raw in enumerate(fh, 1):
            line = raw.rstrip("\n")
            if not line:
                continue
            fields = line.split("\t")
            if len(fields) != 2:
                raise ValueError(f"{path}: line {lineno}: expected 2 tab-separated fields, got {len(fields)}")
            out.append((fields[0], fields[1]))
    return out


def read_parallel(path: str | os.PathLike) -> list[tuple[str, str]]:
    """``source<TAB>target`` sentence pairs (lexicon / classifier training)."""
    return _two_fields(path)


def read_links(path: str | os.PathLike) -> list[tuple[str, str]]:
    """Two tab-separated columns per line (document links, title pairs)."""
    return _two_fields(path)
