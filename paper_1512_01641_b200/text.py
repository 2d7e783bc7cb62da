"""The single tokenizer of the path (text.py:97-104 of the reference).

``tokenize`` lowercases, splits on whitespace and strips ASCII
punctuation from both ends of every token, dropping tokens that become
empty.  It stays on the host: the device only ever sees token ids.
"""

from __future__ import annotations

import string

_PUNCT = string.punctuation


def tokenize(text: str) -> list[str]:
    """Lowercase, split on whitespace, strip surrounding punctuation."""
    return [tok for tok in (raw.strip(_PUNCT) for raw in text.lower().split()) if tok]
