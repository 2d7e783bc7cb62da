"""Similarity model parameters (reference classifier.py:115-184).

The per-cell arithmetic (features -> margin -> logistic) runs on the
device (csrc/score_kernel.cuh).  This module holds the 21 model doubles,
their validation and JSON I/O, and scalar ``margin``/``score_from_margin``
for API compatibility.  ``model_vector`` accepts the reference's own
``SimilarityModel`` objects as well (same attribute names).
"""

from __future__ import annotations

import json
import math
import os
from dataclasses import dataclass
from typing import Sequence

import numpy as np

FEATURE_COUNT = 6
MODEL_FORMAT_VERSION = 1


@dataclass(frozen=True)
class SimilarityModel:
    """Standardised linear classifier plus Platt sigmoid calibration."""

    weights: tuple[float, ...]
    bias: float
    sigmoid_a: float
    sigmoid_b: float
    feature_means: tuple[float, ...]
    feature_scales: tuple[float, ...]

    def __post_init__(self) -> None:
        for name in ("weights", "feature_means", "feature_scales"):
            if len(getattr(self, name)) != FEATURE_COUNT:
                raise ValueError(f"{name} must have length {FEATURE_COUNT}")
        if any(scale <= 0.0 for scale in self.feature_scales):
            raise ValueError("feature scales must be positive")
        if self.sigmoid_a >= 0.0:
            raise ValueError("sigmoid_a must be negative")

    def margin(self, features: Sequence[float]) -> float:
        d = self.bias
        for w, f, m, s in zip(self.weights, features, self.feature_means, self.feature_scales):
            d += w * (f - m) / s
        return d

    def score_from_margin(self, margin: float) -> float:
        z = self.sigmoid_a * margin + self.sigmoid_b
        if z >= 0:
            p = math.exp(-z) / (1.0 + math.exp(-z)) if z < 700 else 0.0
        else:
            p = 1.0 / (1.0 + math.exp(z)) if z > -700 else 1.0
        return min(max(p, 0.0), 1.0)

    def to_dict(self) -> dict:
        return {
            "version": MODEL_FORMAT_VERSION,
            "weights": list(self.weights),
            "bias": self.bias,
            "sigmoid_a": self.sigmoid_a,
            "sigmoid_b": self.sigmoid_b,
            "feature_means": list(self.feature_means),
            "feature_scales": list(self.feature_scales),
        }

    @classmethod
    def from_dict(cls, data: dict) -> "SimilarityModel":
        version = data.get("version")
        if version != MODEL_FORMAT_VERSION:
            raise ValueError(f"unsupported model format version: {version!r}")
        return cls(
            weights=tuple(float(v) for v in data["weights"]),
            bias=float(data["bias"]),
            sigmoid_a=float(data["sigmoid_a"]),
            sigmoid_b=float(data["sigmoid_b"]),
            feature_means=tuple(float(v) for v in data["feature_means"]),
            feature_scales=tuple(float(v) for v in data["feature_scales"]),
        )


def save_model(model: SimilarityModel, path: str | os.PathLike) -> None:
    with open(path, "w", encoding="utf-8") as handle:
        json.dump(model.to_dict(), handle, indent=2, sort_keys=True)
        handle.write("\n")


def load_model(path: str | os.PathLike) -> SimilarityModel:
    with open(path, encoding="utf-8") as handle:
        return SimilarityModel.from_dict(json.load(handle))


def model_vector(model) -> np.ndarray:
    """The 21 doubles in BIMINE_MODEL_DOUBLES order (include/bimine_b200.h)."""
    vec = np.empty(21, dtype=np.float64)
    vec[0:6] = [float(v) for v in model.weights]
    vec[6] = float(model.bias)
    vec[7] = float(model.sigmoid_a)
    vec[8] = float(model.sigmoid_b)
    vec[9:15] = [float(v) for v in model.feature_means]
    vec[15:21] = [float(v) for v in model.feature_scales]
    if len(model.weights) != 6 or len(model.feature_means) != 6 or len(model.feature_scales) != 6:
        raise ValueError(f"model vectors must have length {FEATURE_COUNT}")
    return vec


def similarity(model, source_sentence: str, target_sentence: str, lexicon) -> float:
    """Calibrated translation-likelihood score of one sentence pair
    (classifier.py:357-362): the 1x1 score matrix of the GPU path, so the
    same bits as ``build_score_matrix`` (align.py:102-129)."""
    from .align import build_score_matrix

    try:
        return float(build_score_matrix(model, lexicon, [source_sentence], [target_sentence])[0, 0])
    except ValueError as exc:  # the reference reports profile_sentence's message unprefixed
        msg = str(exc)
        for prefix in ("source sentence 0: ", "target sentence 0: "):
            if msg.startswith(prefix):
                raise ValueError(msg[len(prefix):]) from None
        raise


# any valid model: the features do not depend on it (the kernel also scores)
_FEATURE_MODEL = np.array([0.0] * 6 + [0.0, -1.0, 0.0] + [0.0] * 6 + [1.0] * 6, dtype=np.float64)


def extract_features(source_sentence: str, target_sentence: str, lexicon) -> list[float]:
    """Six-feature description of a sentence pair (classifier.py:100-112):
    token-length ratio (capped at 4), source coverage, target coverage, mean
    best translation probability, char-length ratio (capped at 4), shared
    identical tokens -- computed by the score kernel's features mode
    (bimine_features_batch), the same arithmetic the scores use."""
    from . import engine as E
    from .align import _pack_one

    ctx = E.lexicon_context(lexicon)
    try:
        batch = _pack_one(ctx.vocab, [source_sentence], [target_sentence])
    except ValueError as exc:  # profile_sentence's message, unprefixed
        msg = str(exc)
        for prefix in ("source sentence 0: ", "target sentence 0: "):
            if msg.startswith(prefix):
                raise ValueError(msg[len(prefix):]) from None
        raise
    feats = E.features_host(ctx.on(E.current_device()), _FEATURE_MODEL, batch)
    return [float(v) for v in feats[0]]
