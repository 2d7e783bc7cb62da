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


# Dictionary probabilities of every float class the reference's lexicon
# reader admits (lexicon.py:165-178 keeps any float(field)); the p > 0 rules
# (classifier.py:58,78) drop zero, negative and NaN entries.  The same
# recipe makes the golden fixture (make_golden.py extreme_fixture) and
# drives the CPU and GPU parity tests against it.
EXTREME_VARIANTS = ("fine", "huge", "inf")


def extreme_probabilities(prob: np.ndarray, variant: str, seed: int = 1512) -> np.ndarray:
    rng = np.random.default_rng(seed)
    u = rng.random(prob.size)
    full = rng.random(prob.size)  # full-precision values in [0, 1)
    pick = rng.integers(0, 3, size=prob.size)
    p = prob.astype(np.float64).copy()
    classes = [
        (0.00, 0.10, full),
        (0.10, 0.14, np.array([5e-324, 1e-310, 2.225073858507201e-308])[pick]),  # subnormal
        (0.14, 0.17, np.array([1e-300, 2.2250738585072014e-308, 1e-30])[pick]),  # tiny normal
        (0.17, 0.27, np.full(prob.size, 0.25)),  # ties
        (0.27, 0.31, np.array([1.0, 3.5, 1e10])[pick]),  # >= 1
        (0.31, 0.35, np.array([0.0, -0.5, np.nan])[pick]),  # dropped
    ]
    if variant == "huge":  # sums overflow to +inf
        classes.append((0.35, 0.356, np.array([1e308, 1.5e308, 1.7976931348623157e308])[pick]))
    elif variant == "inf":
        classes.append((0.35, 0.352, np.full(prob.size, np.inf)))
    elif variant != "fine":
        raise ValueError(variant)
    for lo, hi, v in classes:
        sel = (u >= lo) & (u < hi)
        p[sel] = v[sel]
    return p


def extreme_corpora():
    """(name, corpus, pairs) the extreme-probability fixture covers: C1's
    200 x 220 pair (tiled score path) and three C2 pairs (pair_kernel)."""
    from paper_1512_01641_b200 import synth

    return [("c1", synth.make_config(1), [0]), ("c2", synth.make_config(2, n_pairs=3), [0, 1, 2])]
