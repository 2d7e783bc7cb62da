"""Fixture loading shared by the CPU and GPU parity tests."""

from __future__ import annotations

import json
import os
from functools import lru_cache

import numpy as np

from paper_1512_01641_b200.classifier import SimilarityModel, load_model, model_vector
from paper_1512_01641_b200.lexicon import Lexicon
from paper_1512_01641_b200.packing import BatchBuilder, Vocabulary, lexicon_arrays

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _unhex(v):
    if isinstance(v, list):
        return [_unhex(x) for x in v]
    if isinstance(v, str):
        return float.fromhex(v)
    return v


@lru_cache(maxsize=None)
def load_json(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


@lru_cache(maxsize=None)
def load_npz(name):
    with np.load(os.path.join(GOLDEN, name)) as z:
        return {k: z[k] for k in z.files}


def toy_model() -> SimilarityModel:
    d = load_json("toy.json")["model"]
    return SimilarityModel.from_dict({k: (_unhex(v) if k != "version" else v) for k, v in d.items()})


def toy_lexicon() -> Lexicon:
    table = {}
    for s, t, p in load_json("toy.json")["lexicon"]:
        table.setdefault(s, {})[t] = float.fromhex(p)
    return Lexicon(table)


def synth_model() -> SimilarityModel:
    return load_model(os.path.join(GOLDEN, "synth_model.json"))


def pack_pairs(lexicon, pairs):
    """(vocab, COO dictionary arrays, PackedBatch) for [(src_sents, tgt_sents)]."""
    vocab = Vocabulary()
    src, tgt, prob = lexicon_arrays(lexicon.items(), vocab)
    builder = BatchBuilder(vocab)
    for s, t in pairs:
        builder.add_pair(s, t)
    return vocab, (src, tgt, prob), builder.build()


def toy_pairs():
    return [(p["source"], p["target"]) for p in load_json("toy.json")["pairs"]]


def toy_sims():
    z = load_npz("toy_sims.npz")
    return [z[f"sim{k}"] for k in range(len(z))]


def nw_family(name):
    z = load_npz("nw_golden.npz")
    codes, offs = z[f"{name}_codes"], z[f"{name}_offs"]
    return [
        (codes[offs[k] : offs[k + 1]], z[f"{name}_scores"][k], tuple(z[f"{name}_shapes"][k]), z[f"{name}_gaps"][k])
        for k in range(len(offs) - 1)
    ]


def nw_family_sims(name):
    """Regenerate the matrices of a reference instance family from its seed
    (same generators as tests/golden/make_golden.py:nw_fixture)."""
    if name.startswith("exact_"):
        rng = np.random.default_rng(int(name.split("_")[1]))
        for _ in range(200):
            n = int(rng.integers(1, 8))
            m = int(rng.integers(1, 8))
            s = rng.integers(0, 3, size=n)
            t = rng.integers(0, 3, size=m)
            yield (s[:, None] == t[None, :]).astype(np.float64)
    elif name.startswith("float_"):
        seed = int(name.split("_")[1])
        count, lo, hi = {7: (20, 1, 12), 11: (30, 1, 15), 29: (25, 1, 80)}[seed]
        rng = np.random.default_rng(seed)
        for _ in range(count):
            sim = rng.random((int(rng.integers(lo, hi)), int(rng.integers(lo, hi))))
            rng.uniform(0, 3.0)
            yield sim
    elif name == "acceptance_2002":
        rng = np.random.default_rng(2002)
        for _ in range(500):
            n = int(rng.integers(1, 201))
            m = int(rng.integers(1, 201))
            sim = rng.random((n, m))
            rng.uniform(0.0, 3.0)
            yield sim
    elif name.startswith("ties_"):
        rng = np.random.default_rng(int(name.split("_")[1]))
        for k in range(200):
            n = int(rng.integers(1, 40))
            m = int(rng.integers(1, 40))
            levels = 2 if k % 2 else 4
            sim = rng.integers(0, levels, size=(n, m)) / (levels - 1)
            rng.integers(0, 3)
            yield sim
    else:
        raise KeyError(name)


NW_FAMILIES = ["exact_2024", "exact_1001", "float_7", "float_11", "float_29", "acceptance_2002", "ties_5"]
NW_MISMATCH, NW_BONUS = -1.0, 1.0


def codes_of(steps) -> np.ndarray:
    return np.asarray(steps, dtype=np.uint8)


def match_triples(rows):
    return [(float(s), int(i), int(j)) for s, i, j in rows]
