"""Document-pair inputs of the mining API (reference corpus.py:21-51).

Only the two value types the hot path consumes live here; corpus file
I/O is outside the path.  Functions in
``align`` accept any object with the same attributes (duck typing), so
the reference's own ``bimine.corpus.DocumentPair`` instances work too.
"""

from __future__ import annotations

from dataclasses import dataclass


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
