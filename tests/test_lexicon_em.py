"""Lexicon EM (reference lexicon.py:60-120).

Golden tables were produced by the reference's own build_lexicon
(tests/golden/make_golden.py lexicon).  CPU: the oracle restatement is
pinned to them.  GPU: the product (rounds in csrc/lexicon_em.cuh) equals
them and the oracle bit for bit, and raises the reference's errors.
"""

import json
import os

import numpy as np
import pytest

import oracle

HERE = os.path.dirname(os.path.abspath(__file__))


def _golden():
    with open(os.path.join(HERE, "golden", "lexicon_em.json")) as fh:
        g = json.load(fh)
    for run in g["runs"]:
        run["want"] = {s: {t: float.fromhex(h) for t, h in row.items()} for s, row in run["table"].items()}
    return g


def _pairs(g, name):
    return [tuple(x) for x in g["inputs"][name]]


def test_oracle_restatement_matches_reference_tables():
    g = _golden()
    for run in g["runs"]:
        got = oracle.build_lexicon(_pairs(g, run["name"]), run["iterations"], run["prune"])
        assert got == run["want"], (run["name"], run["iterations"])


def test_oracle_errors():
    with pytest.raises(ValueError, match="no training pairs"):
        oracle.build_lexicon([], 3)
    with pytest.raises(ValueError, match="iterations must be >= 1"):
        oracle.build_lexicon([("a", "b")], 0)
    with pytest.raises(ValueError, match="no training pairs"):
        oracle.build_lexicon([("...", "b"), ("a", "!!")], 2)


@pytest.mark.gpu
def test_gpu_build_lexicon_matches_reference_tables():
    from paper_1512_01641_b200.lexicon import build_lexicon

    g = _golden()
    for run in g["runs"]:
        lex = build_lexicon(_pairs(g, run["name"]), run["iterations"], prune_threshold=run["prune"])
        assert lex._table == run["want"], (run["name"], run["iterations"])


@pytest.mark.gpu
def test_gpu_build_lexicon_matches_oracle_on_a_larger_corpus():
    from paper_1512_01641_b200 import synth
    from paper_1512_01641_b200.lexicon import build_lexicon

    d = synth.make_dictionary(np.random.default_rng(91), 2000)
    corpus = synth.make_corpus(92, 30, 2000, dictionary=d)
    par = []
    for p in range(30):
        src, tgt = corpus.pair_sentences(p)
        par += [(src[i], tgt[j]) for i, j in corpus.reference[p]]
        par.append((src[-1], tgt[0]))
    for iters, prune in [(4, 1e-4), (1, 0.0)]:
        assert build_lexicon(par, iters, prune_threshold=prune)._table == oracle.build_lexicon(par, iters, prune)


@pytest.mark.gpu
def test_gpu_build_lexicon_errors():
    from paper_1512_01641_b200.lexicon import build_lexicon

    with pytest.raises(ValueError, match="no training pairs"):
        build_lexicon([], 3)
    with pytest.raises(ValueError, match="iterations must be >= 1"):
        build_lexicon([("a", "b")], 0)
    with pytest.raises(ValueError, match="no training pairs"):
        build_lexicon([("...", "b")], 2)


def test_py_sum_is_the_interpreters_sum():
    """The restated float sum is bit-identical to this interpreter's sum()
    (Neumaier-compensated since CPython 3.12), incl. -0.0, huge ranges, inf."""
    import random

    rng = random.Random(11)
    cases = [[], [-0.0], [0.0, -0.0], [1e308, 1e308, -1e308], [float("inf"), 1.0], [1.0, 1e100, 1.0, -1e100]]
    for _ in range(5000):
        cases.append([rng.uniform(-1, 1) * 10.0 ** rng.randint(-30, 30) for _ in range(rng.randint(1, 20))])
    for xs in cases:
        assert repr(oracle.py_sum(xs)) == repr(sum(xs)), xs
