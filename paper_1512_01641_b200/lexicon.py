"""Bilingual dictionary (reference lexicon.py:22-59, 153-178).

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
from typing import Iterator, Mapping


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
