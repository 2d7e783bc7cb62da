"""Generate the golden fixtures by running the REFERENCE implementation.

Run in the build container, where /root/reference exists:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports the reference package (pkg/src/bimine) and its test fixture
recipes (pkg/tests/conftest.py, oracles.py) read-only, evaluates them on
seeded inputs and writes their outputs here.  The fixtures are what the
CPU oracle (oracle/) and the CUDA path are pinned against on machines
without the reference (the GPU box).  Nothing here is imported at run
time by the product.
"""

from __future__ import annotations

import json
import math
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))

sys.dont_write_bytecode = True
os.environ.setdefault("BIMINE_PURE_PYTHON", "")
sys.path[:0] = [REF_SRC, REF_TESTS, REPO]

from bimine import align as ref_align  # noqa: E402
from bimine.align import (  # noqa: E402
    GapSource,
    Match,
    MiningConfig,
    build_score_matrix,
    filter_by_threshold,
    mine_document_pair,
    nw_align,
)
from bimine.classifier import make_negative_pairs, train_classifier  # noqa: E402
from bimine.corpus import Document, DocumentPair  # noqa: E402
from bimine.lexicon import Lexicon, build_lexicon  # noqa: E402
from bimine.tuning import TuningSample, alignment_agreement, tune  # noqa: E402

import conftest as ref_conftest  # noqa: E402

from paper_1512_01641_b200 import synth  # noqa: E402


def step_codes(alignment) -> list[int]:
    return [0 if isinstance(s, Match) else 1 if isinstance(s, GapSource) else 2 for s in alignment.steps]


def rows_json(rows):
    return [[float(score).hex(), src, tgt] for score, src, tgt in rows]


def toy_fixture():
    corpus = ref_conftest.make_parallel_sentences(np.random.default_rng(1234), 60)
    lexicon = build_lexicon(corpus, 10)
    rng = np.random.default_rng(4321)
    positives = ref_conftest.make_parallel_sentences(rng, 80)
    negatives = make_negative_pairs(positives, 99)
    model = train_classifier(positives, negatives, lexicon, epochs=12, seed=7)

    pairs = []
    for seed, name, true_pairs, noise in [
        (59, "alpha", 6, 2), (61, "beta", 6, 2), (53, "probe", 5, 0),
        (67, "topic-0", 6, 2), (71, "good", 6, 2), (83, "few-0", 6, 2),
        (101, "wide", 12, 9), (102, "tall", 15, 1),
    ]:
        pair, reference = ref_conftest.make_mining_pair(np.random.default_rng(seed), name, true_pairs, noise)
        pairs.append((pair, reference))
    # hand-written edge pairs: single sentences, unrelated documents,
    # punctuation, repeated tokens, mixed case
    edge = [
        ("single", ("domo kato",), ("house cat",)),
        ("unrelated", ("domo kato hundo",), ("zork blip quux",)),
        ("punct", ("Domo, kato!", "...libro... akvo;", "domo domo domo kato"),
         ("House cat.", "book -- water", "house house cat", "(dog)")),
        ("shared", ("zork domo zork", "blip"), ("zork house", "blip blip zork", "cat")),
    ]
    for name, src, tgt in edge:
        pair = DocumentPair(
            topic_id=name,
            source=Document(id=name + "-s", lang="eo", title=name, sentences=src),
            target=Document(id=name + "-t", lang="en", title=name, sentences=tgt),
        )
        pairs.append((pair, []))

    out = {
        "lexicon": [[s, t, float(p).hex()] for s, t, p in lexicon.items()],
        "model": {k: ([float(x).hex() for x in v] if isinstance(v, (list, tuple)) else (float(v).hex() if isinstance(v, float) else v))
                  for k, v in model.to_dict().items()},
        "pairs": [],
    }
    sims = {}
    for k, (pair, reference) in enumerate(pairs):
        sim = build_score_matrix(model, lexicon, pair.source.sentences, pair.target.sentences)
        sims[f"sim{k}"] = sim
        entry = {
            "topic_id": pair.topic_id,
            "source": list(pair.source.sentences),
            "target": list(pair.target.sentences),
            "reference": [list(x) for x in reference],
        }
        for cfg_name, cfg in [("default", MiningConfig()), ("strict", MiningConfig(threshold=0.8, gap_penalty=0.5)),
                              ("loose", MiningConfig(threshold=0.0, gap_penalty=3.0, match_bonus=2.0, mismatch_cost=-0.5))]:
            al = nw_align(sim, cfg)
            entry[cfg_name] = {
                "steps": step_codes(al),
                "score": float(al.score).hex(),
                "rows": rows_json(mine_document_pair(model, lexicon, pair, cfg, engine="nw")),
                "indices": [[float(s).hex(), i, j] for s, i, j in filter_by_threshold(sim, al, cfg.threshold)],
            }
        out["pairs"].append(entry)
    # an untokenizable sentence: the reference's error text
    try:
        build_score_matrix(model, lexicon, ["domo"], ["house", "..."])
    except ValueError as exc:
        out["error_untokenizable"] = str(exc)
    bad = DocumentPair(
        topic_id="bad",
        source=Document(id="b1", lang="eo", title="bad", sentences=("...",)),
        target=Document(id="b2", lang="en", title="bad", sentences=("house",)),
    )
    out["mine_corpus_failures"] = [list(f) for f in ref_align.mine_corpus(
        model, lexicon, [pairs[0][0], bad], MiningConfig(), engine="nw").failures]
    with open(os.path.join(HERE, "toy.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    np.savez_compressed(os.path.join(HERE, "toy_sims.npz"), **sims)
    print("toy fixture:", len(pairs), "pairs")


def synth_model_fixture():
    """Classifier for the synthetic benchmark data, trained by the
    reference's own train_classifier."""
    corpus = synth.make_config(2, n_pairs=80)
    positives = []
    for p, ref in enumerate(corpus.reference):
        src, tgt = corpus.pair_sentences(p)
        positives.extend((src[i], tgt[j]) for i, j in ref)
        if len(positives) >= 2000:
            break
    positives = positives[:2000]
    lexicon = Lexicon(corpus.dictionary.table())
    negatives = make_negative_pairs(positives, 99)
    model = train_classifier(positives, negatives, lexicon, epochs=12, seed=7)
    with open(os.path.join(HERE, "synth_model.json"), "w") as fh:
        json.dump(model.to_dict(), fh, indent=2, sort_keys=True)
        fh.write("\n")
    print("synth model:", model)
    return model, lexicon


def synth_fixtures(model, lexicon_c2):
    def run(corpus, lexicon, pairs, name):
        sims, steps, scores, rows = {}, [], [], []
        for p in pairs:
            src, tgt = corpus.pair_sentences(p)
            sim = build_score_matrix(model, lexicon, src, tgt)
            sims[f"sim{p}"] = sim
            al = nw_align(sim, MiningConfig())
            steps.append(step_codes(al))
            scores.append(float(al.score).hex())
            rows.append([[float(s).hex(), i, j] for s, i, j in filter_by_threshold(sim, al, 0.5)])
        np.savez_compressed(os.path.join(HERE, f"{name}_sims.npz"), **sims)
        with open(os.path.join(HERE, f"{name}.json"), "w") as fh:
            json.dump({"pairs": list(pairs), "steps": steps, "scores": scores, "indices": rows}, fh)
        print(name, "pairs", list(pairs), "matches", [len(r) for r in rows])

    c1 = synth.make_config(1)
    run(c1, Lexicon(c1.dictionary.table()), [0], "synth_c1")
    c2 = synth.make_config(2, n_pairs=12)
    run(c2, lexicon_c2, list(range(12)), "synth_c2")


def extreme_fixture():
    """Reference score matrices and mined rows with dictionary
    probabilities of every float class (tests/helpers.py
    extreme_probabilities): subnormal, tied, > 1, dropped (zero, negative,
    NaN), overflowing and infinite values."""
    import dataclasses

    sys.path.insert(0, os.path.dirname(HERE))
    import helpers as H
    from bimine.classifier import load_model

    model = load_model(os.path.join(HERE, "synth_model.json"))
    sims, out = {}, {}
    for variant in H.EXTREME_VARIANTS:
        for cname, corpus, pairs in H.extreme_corpora():
            d = corpus.dictionary
            d = dataclasses.replace(d, prob=H.extreme_probabilities(d.prob, variant))
            lexicon = Lexicon(d.table())
            for p in pairs:
                src, tgt = corpus.pair_sentences(p)
                sim = build_score_matrix(model, lexicon, src, tgt)
                key = f"{variant}_{cname}_{p}"
                sims[key] = sim
                al = nw_align(sim, MiningConfig())
                out[key] = {"steps": step_codes(al), "score": float(al.score).hex(),
                            "indices": [[float(s).hex(), i, j] for s, i, j in filter_by_threshold(sim, al, 0.5)]}
                print(key, sim.shape, "distinct scores", len(np.unique(sim)), "matches", len(out[key]["indices"]))
    np.savez_compressed(os.path.join(HERE, "extreme_sims.npz"), **sims)
    with open(os.path.join(HERE, "extreme.json"), "w") as fh:
        json.dump(out, fh)


def nw_fixture():
    """Reference nw_align outputs on the reference tests' own instance
    families (test_align.py:38-43,68-115; test_acceptance.py:56-110)."""
    families = {}

    def exact_instances(seed, count, max_len=7):
        rng = np.random.default_rng(seed)
        for _ in range(count):
            n = int(rng.integers(1, max_len + 1))
            m = int(rng.integers(1, max_len + 1))
            s = rng.integers(0, 3, size=n)
            t = rng.integers(0, 3, size=m)
            yield (s[:, None] == t[None, :]).astype(np.float64), MiningConfig(threshold=0.0, gap_penalty=2.0)

    def float_instances(seed, count, lo, hi, gap_hi=3.0):
        rng = np.random.default_rng(seed)
        for _ in range(count):
            sim = rng.random((int(rng.integers(lo, hi)), int(rng.integers(lo, hi))))
            yield sim, MiningConfig(gap_penalty=float(rng.uniform(0, gap_hi)))

    def acceptance_instances():
        rng = np.random.default_rng(2002)
        for _ in range(500):
            n = int(rng.integers(1, 201))
            m = int(rng.integers(1, 201))
            sim = rng.random((n, m))
            yield sim, MiningConfig(gap_penalty=float(rng.uniform(0.0, 3.0)))

    def tie_instances(seed, count):
        # 4-level and 0/1 matrices with gap 0 and integer gaps: tie heavy
        rng = np.random.default_rng(seed)
        for k in range(count):
            n = int(rng.integers(1, 40))
            m = int(rng.integers(1, 40))
            levels = 2 if k % 2 else 4
            sim = rng.integers(0, levels, size=(n, m)) / (levels - 1)
            gap = float(rng.integers(0, 3)) * 0.5
            yield sim, MiningConfig(gap_penalty=gap)

    gens = {
        "exact_2024": exact_instances(2024, 200),
        "exact_1001": exact_instances(1001, 200),
        "float_7": float_instances(7, 20, 1, 12),
        "float_11": float_instances(11, 30, 1, 15),
        "float_29": float_instances(29, 25, 1, 80),
        "acceptance_2002": acceptance_instances(),
        "ties_5": tie_instances(5, 200),
    }
    out = {}
    for name, gen in gens.items():
        codes, offs, scores, shapes, gaps = [], [0], [], [], []
        for sim, cfg in gen:
            al = nw_align(sim, cfg)
            c = step_codes(al)
            codes.extend(c)
            offs.append(len(codes))
            scores.append(al.score)
            shapes.append(sim.shape)
            gaps.append(cfg.gap_penalty)
        out[f"{name}_codes"] = np.asarray(codes, dtype=np.uint8)
        out[f"{name}_offs"] = np.asarray(offs, dtype=np.int64)
        out[f"{name}_scores"] = np.asarray(scores, dtype=np.float64)
        out[f"{name}_shapes"] = np.asarray(shapes, dtype=np.int64)
        out[f"{name}_gaps"] = np.asarray(gaps, dtype=np.float64)
    np.savez_compressed(os.path.join(HERE, "nw_golden.npz"), **out)
    print("nw fixture families:", list(gens))


def exp_fixture():
    """math.exp on the logistic's argument range (classifier.py:145-147)
    plus the branch edges of glibc's exp."""
    rng = np.random.default_rng(31337)
    x = np.concatenate([
        -rng.uniform(0, 700, 20_000),
        -rng.uniform(0, 40, 20_000),
        -rng.uniform(0, 1e-3, 2_000),
        -np.exp(rng.uniform(np.log(1e-300), np.log(1e-10), 2_000)),
        -rng.uniform(511, 513, 2_000),
        np.array([0.0, -0.0, -1e-300, -5e-324, -2 ** -54, -2 ** -53, -699.999, -700.0, -512.0, -511.9999999,
                  -708.0, -708.4, -709.0, -745.0, -744.44, -1.0, -0.5, -math.log(2), -1e-17]),
    ])
    y = np.array([math.exp(float(v)) for v in x], dtype=np.float64)
    np.savez_compressed(os.path.join(HERE, "exp_golden.npz"), x=x, y=y)
    print("exp fixture:", x.size)


def tuning_fixture():
    """tune() (tuning.py:92-153) on synthetic C4-shaped samples whose
    reference alignments are the generator's true translation indices."""
    from bimine.classifier import load_model
    model = load_model(os.path.join(HERE, "synth_model.json"))
    corpus = synth.make_config(4, n_pairs=6)
    lexicon = Lexicon(corpus.dictionary.table())
    samples = []
    for p in range(6):
        src, tgt = corpus.pair_sentences(p)
        pair = DocumentPair(
            topic_id=f"tune-{p}",
            source=Document(id=f"tune-{p}-s", lang="pl", title=str(p), sentences=tuple(src)),
            target=Document(id=f"tune-{p}-t", lang="en", title=str(p), sentences=tuple(tgt)),
        )
        samples.append(TuningSample(pair=pair, reference=tuple(tuple(r) for r in corpus.reference[p])))
    result = tune(model, lexicon, samples, budget=16, seed=5, engine="nw")
    agreement_kats = []
    kat_rng = np.random.default_rng(17)
    for _ in range(50):
        ref = sorted({(int(a), int(a) + int(b)) for a, b in zip(kat_rng.integers(0, 12, 6), kat_rng.integers(0, 3, 6))})
        cand = sorted({(int(a), int(a) + int(b)) for a, b in zip(kat_rng.integers(0, 12, 6), kat_rng.integers(0, 3, 6))})
        agreement_kats.append([ref, cand, alignment_agreement(cand, ref)])
    out = {
        "config": 4, "n_pairs": 6,
        "budget": 16, "seed": 5,
        "result": {
            "threshold": float(result.threshold).hex(), "gap_penalty": float(result.gap_penalty).hex(),
            "agreement": float(result.agreement).hex(), "trials": result.trials,
            "per_sample": [float(v).hex() for v in result.per_sample],
            "default_agreement": float(result.default_agreement).hex(),
        },
        "agreement_kats": [[[list(x) for x in r], [list(x) for x in c], float(v).hex()] for r, c, v in agreement_kats],
    }
    with open(os.path.join(HERE, "tune_golden.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print("tuning fixture:", result)


def features_fixture():
    """extract_features (classifier.py:100-112) by the reference on every
    cell of the toy pairs (toy.json's lexicon) and on hand-picked edge
    pairs: ratio caps at 4, no coverage, identical sentences, repeated and
    shared tokens."""
    from bimine.classifier import extract_features

    with open(os.path.join(HERE, "toy.json")) as fh:
        toy = json.load(fh)
    table = {}
    for s, t, p in toy["lexicon"]:
        table.setdefault(s, {})[t] = float.fromhex(p)
    lex = Lexicon(table)
    cells = []
    for pair in toy["pairs"]:
        for a in pair["source"]:
            for b in pair["target"]:
                cells.append([a, b, [float(v).hex() for v in extract_features(a, b, lex)]])
    edge = [("domo kato hundo domo kato hundo domo kato hundo", "house"), ("x", "a b c d e f g h i j"),
            ("zork blip", "quux flub"), ("domo domo domo", "house house"), ("Domo, KATO!", "domo kato"),
            ("libro floro", "libro book flower"), ("a", "a")]
    for a, b in edge:
        cells.append([a, b, [float(v).hex() for v in extract_features(a, b, lex)]])
    with open(os.path.join(HERE, "features_golden.json"), "w") as fh:
        json.dump({"cells": cells}, fh, indent=0)
    print("features fixture:", len(cells), "cells")


def lexicon_em_fixture():
    """build_lexicon (lexicon.py:60-120) run by the reference on (a) the
    parallel corpus its own test fixtures train on (conftest.py) and (b) a
    synthetic corpus with repeated tokens, mixed case, punctuation, a pair
    with an empty side and unrelated pairs; several round counts and prune
    thresholds.  Probabilities are stored as float.hex()."""
    cases = []
    toy = ref_conftest.make_parallel_sentences(np.random.default_rng(1234), 60)
    cases.append(("toy", toy, [(10, 1e-4), (1, 1e-4), (3, 0.0)]))
    rng = np.random.default_rng(555)
    d = synth.make_dictionary(rng, 300)
    corpus = synth.make_corpus(556, 6, 300, dictionary=d)
    par = []
    for p in range(6):
        src, tgt = corpus.pair_sentences(p)
        for i, j in corpus.reference[p]:
            par.append((src[i], tgt[j]))
        par.append((src[0], tgt[-1]))  # an unrelated pair
    par += [("Domo domo, KATO!", "house House cat"), ("...", "nothing"), ("alpha beta alpha", "gamma gamma delta")]
    cases.append(("synth", par, [(5, 1e-4), (8, 0.05)]))
    out = []
    for name, parallel, runs in cases:
        for iters, prune in runs:
            lex = build_lexicon(parallel, iters, prune_threshold=prune)
            table = {s: {t: float(p).hex() for t, p in row.items()} for s, row in lex._table.items()}
            out.append({"name": name, "iterations": iters, "prune": prune, "table": table})
        out_inputs = {name: [list(x) for x in parallel] for name, parallel, _ in cases}
    with open(os.path.join(HERE, "lexicon_em.json"), "w") as fh:
        json.dump({"inputs": out_inputs, "runs": out}, fh, indent=0)
    print("lexicon fixture:", [(r["name"], r["iterations"], len(r["table"])) for r in out])


def cli_fixture():
    """The reference CLI's `mine` and `tune` (cli.py:129-230) on a small
    synthetic corpus directory: the bitext bytes, printed lines, exit codes
    and tuning report a file-level drop-in must reproduce.  The corpus has a
    topic id with a backslash, a title with a tab (field escaping) and one
    pair with an untokenizable sentence (failure path, exit status 1)."""
    import contextlib
    import io
    import shutil
    import tempfile

    from bimine import cli as ref_cli
    from bimine.corpus import save_corpus
    from bimine.lexicon import write_lexicon

    out_dir = os.path.join(HERE, "cli")
    shutil.rmtree(out_dir, ignore_errors=True)
    os.makedirs(out_dir)
    d = synth.make_dictionary(np.random.default_rng(777), 1000)
    corpus = synth.make_corpus(778, 10, 1000, dictionary=d)
    pairs = []
    for p in range(10):
        src, tgt = corpus.pair_sentences(p)
        topic = f"cli-{p}" if p != 3 else "cli\\3"
        title = f"title {p}" if p != 5 else "tab\there"
        if p == 7:
            tgt = tgt[:4] + ["..."] + tgt[4:]
        pairs.append(DocumentPair(
            topic_id=topic,
            source=Document(id=f"s{p}", lang="pl", title=title, sentences=tuple(src)),
            target=Document(id=f"t{p}", lang="en", title=title, sentences=tuple(tgt)),
        ))
    corpus_dir = os.path.join(out_dir, "corpus")
    save_corpus(pairs, corpus_dir)
    lex_path = os.path.join(out_dir, "lexicon.tsv")
    write_lexicon(Lexicon(d.table()), lex_path)
    model_path = os.path.join(HERE, "synth_model.json")
    with open(os.path.join(out_dir, "reference.tsv"), "w", encoding="utf-8") as fh:
        for p in (0, 1, 2, 4):
            for i, j in corpus.reference[p]:
                fh.write(f"{pairs[p].topic_id}\t{i}\t{j}\n")

    def run(argv):
        so, se = io.StringIO(), io.StringIO()
        with contextlib.redirect_stdout(so), contextlib.redirect_stderr(se):
            rc = ref_cli.main(argv)
        return rc, so.getvalue(), se.getvalue()

    expect = {}
    with tempfile.TemporaryDirectory() as tmp:
        for name, extra in (("default", []), ("strict", ["--threshold", "0.8", "--gap-penalty", "1.5"])):
            out = os.path.join(tmp, f"mined_{name}.tsv")
            rc, so, se = run(["mine", corpus_dir, model_path, lex_path, out, *extra])
            shutil.copy(out, os.path.join(out_dir, f"mined_{name}.tsv"))
            expect[f"mine_{name}"] = {"argv": extra, "rc": rc, "stdout": so, "stderr": se}
        rep = os.path.join(tmp, "report.json")
        good = os.path.join(tmp, "good")
        save_corpus([p for k, p in enumerate(pairs) if k != 7], good)
        rc, so, se = run(["tune", good, model_path, lex_path, os.path.join(out_dir, "reference.tsv"),
                          "--budget", "8", "--seed", "3", "--out", rep])
        with open(rep) as fh:
            expect["tune"] = {"rc": rc, "stdout": so, "stderr": se, "report": json.load(fh)}
    # `dict`: EM lexicon from a parallel file, merged with single-token titles
    par = []
    for p in range(4):
        src, tgt = corpus.pair_sentences(p)
        par += [(src[i], tgt[j]) for i, j in corpus.reference[p]]
    with open(os.path.join(out_dir, "parallel.tsv"), "w", encoding="utf-8") as fh:
        fh.writelines(f"{a}\t{b}\n" for a, b in par)
    words = d.words(np.arange(20))  # source words s0..s19
    twords = d.words(d.n_words + np.arange(20))  # target words t0..t19
    with open(os.path.join(out_dir, "titles.tsv"), "w", encoding="utf-8") as fh:
        for k in range(20):
            fh.write(f"{words[k]}\t{twords[k]}\n")
        fh.write("two words\tone\n")
        fh.write("...\tx\n")
    with tempfile.TemporaryDirectory() as tmp:
        out = os.path.join(tmp, "lex.tsv")
        rc, so, se = run(["dict", os.path.join(out_dir, "parallel.tsv"), out,
                          "--titles", os.path.join(out_dir, "titles.tsv")])
        shutil.copy(out, os.path.join(out_dir, "dict_lexicon.tsv"))
        expect["dict"] = {"rc": rc, "stdout": so.replace(out, "<OUT>"), "stderr": se}
    with open(os.path.join(out_dir, "expect.json"), "w") as fh:
        json.dump(expect, fh, indent=1)
    print("cli fixture:", {k: (v["rc"], v["stdout"].strip()[:80]) for k, v in expect.items()})


if __name__ == "__main__":
    which = sys.argv[1:] or ["toy", "synth", "extreme", "nw", "exp", "tune", "cli", "lexicon", "features"]
    if "cli" in which:
        cli_fixture()
    if "lexicon" in which:
        lexicon_em_fixture()
    if "features" in which:
        features_fixture()
    if "toy" in which:
        toy_fixture()
    if "synth" in which:
        model, lex = synth_model_fixture()
        synth_fixtures(model, lex)
    if "nw" in which:
        nw_fixture()
    if "extreme" in which:
        extreme_fixture()
    if "exp" in which:
        exp_fixture()
    if "tune" in which:
        tuning_fixture()
