"""Pin the CPU oracle (oracle/bimine_oracle.c) to the reference's outputs.

The fixtures in tests/golden/ were produced by running the reference
package itself (tests/golden/make_golden.py).  Everything here is CPU
only; the same fixtures pin the CUDA path in test_gpu_parity.py.
"""

import numpy as np
import pytest

import oracle
import helpers as H
from paper_1512_01641_b200 import synth
from paper_1512_01641_b200.classifier import model_vector


@pytest.fixture(scope="module", autouse=True)
def _build_oracle():
    oracle.build()


def _toy_batch():
    lex = H.toy_lexicon()
    vocab, coo, batch = H.pack_pairs(lex, H.toy_pairs())
    return oracle.OracleDict(*coo), batch


def test_toy_score_matrices_bit_exact():
    d, batch = _toy_batch()
    sim = oracle.score_batch(d, model_vector(H.toy_model()), batch)
    for p, ref in enumerate(H.toy_sims()):
        n, m = ref.shape
        got = sim[batch.pair_sim_off[p] : batch.pair_sim_off[p] + n * m].reshape(n, m)
        assert np.array_equal(got.view(np.uint64), ref.view(np.uint64)), f"pair {p}"


@pytest.mark.parametrize("cfg", ["default", "strict", "loose"])
def test_toy_alignments_and_filter(cfg):
    params = {
        "default": dict(gap=2.0, threshold=0.5, mismatch=-1.0, bonus=1.0),
        "strict": dict(gap=0.5, threshold=0.8, mismatch=-1.0, bonus=1.0),
        "loose": dict(gap=3.0, threshold=0.0, mismatch=-0.5, bonus=2.0),
    }[cfg]
    fx = H.load_json("toy.json")["pairs"]
    for p, ref in enumerate(H.toy_sims()):
        codes, si, sj, score = oracle.nw_align(ref, params["mismatch"], params["bonus"], params["gap"])
        assert codes.tolist() == fx[p][cfg]["steps"]
        assert float(score).hex() == fx[p][cfg]["score"]
    d, batch = _toy_batch()
    counts, per_pair = oracle.mine_batch(d, model_vector(H.toy_model()), batch, **params)
    for p in range(batch.n_pairs):
        want = [(float.fromhex(s), i, j) for s, i, j in fx[p][cfg]["indices"]]
        got = [(float(r["score"]), int(r["i"]), int(r["j"])) for r in per_pair[p]]
        assert got == want, f"pair {p}"


@pytest.mark.parametrize("family", H.NW_FAMILIES)
def test_nw_reference_families(family):
    for sim, (codes, score, shape, gap) in zip(H.nw_family_sims(family), H.nw_family(family)):
        assert sim.shape == shape
        got, _, _, got_score = oracle.nw_align(sim, H.NW_MISMATCH, H.NW_BONUS, float(gap))
        assert np.array_equal(got, codes)
        assert got_score == score or (np.isnan(got_score) and np.isnan(score))


def test_nw_table_matches_reference_nwcore():
    """The oracle fill is the reference's own compiled _nwcore fill, bit for bit."""
    nwcore = oracle.reference_nwcore()
    if nwcore is None:
        pytest.skip("oracle/_ref not built (reference sources absent)")
    rng = np.random.default_rng(404)
    for _ in range(30):
        sim = rng.random((int(rng.integers(1, 90)), int(rng.integers(1, 90))))
        gap = float(rng.uniform(0, 3))
        want = oracle.nw_table(sim, -1.0, 1.0, gap)
        dp = np.empty_like(want)
        dp[0, :] = -gap * np.arange(sim.shape[1] + 1, dtype=np.float64)
        dp[1:, 0] = -gap * np.arange(1, sim.shape[0] + 1, dtype=np.float64)
        nwcore.nw_fill(dp, sim, -1.0, 1.0, gap)
        assert np.array_equal(dp.view(np.uint64), want.view(np.uint64))
        dp2 = dp.copy()
        dp2[1:, 1:] = 0
        nwcore.nw_fill_wavefront(dp2, sim, -1.0, 1.0, gap, 4)
        assert np.array_equal(dp2.view(np.uint64), want.view(np.uint64))


def test_synthetic_pairs_bit_exact():
    model = model_vector(H.synth_model())
    for name, corpus in [("synth_c1", synth.make_config(1)), ("synth_c2", synth.make_config(2, n_pairs=12))]:
        fx = H.load_json(f"{name}.json")
        sims = H.load_npz(f"{name}_sims.npz")
        d = oracle.OracleDict(corpus.dictionary.src, corpus.dictionary.tgt, corpus.dictionary.prob)
        sub = corpus.batch.select(fx["pairs"])
        sim = oracle.score_batch(d, model, sub)
        counts, per_pair = oracle.mine_batch(d, model, sub)
        for k, p in enumerate(fx["pairs"]):
            ref = sims[f"sim{p}"]
            n, m = ref.shape
            got = sim[sub.pair_sim_off[k] : sub.pair_sim_off[k] + n * m].reshape(n, m)
            assert np.array_equal(got.view(np.uint64), ref.view(np.uint64)), f"{name} pair {p}"
            want = [(float.fromhex(s), i, j) for s, i, j in fx["indices"][k]]
            assert [(float(r["score"]), int(r["i"]), int(r["j"])) for r in per_pair[k]] == want


def test_synthetic_strings_and_ids_agree():
    """Packing the generator's strings through the host tokenizer gives the
    same score matrices as the generator's own ids (id renaming invariance)."""
    corpus = synth.make_config(2, n_pairs=3)
    from paper_1512_01641_b200.lexicon import Lexicon

    lex = Lexicon(corpus.dictionary.table())
    pairs = [corpus.pair_sentences(p) for p in range(3)]
    _, coo, batch = H.pack_pairs(lex, pairs)
    model = model_vector(H.synth_model())
    a = oracle.score_batch(oracle.OracleDict(*coo), model, batch)
    b = oracle.score_batch(oracle.OracleDict(corpus.dictionary.src, corpus.dictionary.tgt, corpus.dictionary.prob), model, corpus.batch)
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
    assert np.array_equal(batch.sent_chars, corpus.batch.sent_chars)
    assert np.array_equal(batch.sent_uniq, corpus.batch.sent_uniq)


def test_libm_exp_matches_golden():
    """The host's math.exp (glibc, FMA variant) reproduces the fixture made
    where the reference ran; the GPU exp is pinned to the same fixture."""
    z = H.load_npz("exp_golden.npz")
    y = oracle.exp_array(z["x"])
    assert np.array_equal(y.view(np.uint64), z["y"].view(np.uint64))


def test_extreme_probabilities_bit_exact():
    """Dictionary probabilities of every float class (subnormal, tied, > 1,
    dropped zero/negative/NaN, sums overflowing to inf, +inf): the oracle's
    score matrices and mined rows equal the reference's (extreme.json)."""
    model = model_vector(H.synth_model())
    fx = H.load_json("extreme.json")
    sims = H.load_npz("extreme_sims.npz")
    for variant in H.EXTREME_VARIANTS:
        for cname, corpus, pairs in H.extreme_corpora():
            d = corpus.dictionary
            od = oracle.OracleDict(d.src, d.tgt, H.extreme_probabilities(d.prob, variant))
            sub = corpus.batch.select(pairs)
            sim = oracle.score_batch(od, model, sub)
            counts, per_pair = oracle.mine_batch(od, model, sub)
            for k, p in enumerate(pairs):
                key = f"{variant}_{cname}_{p}"
                ref = sims[key]
                n, m = ref.shape
                got = sim[sub.pair_sim_off[k] : sub.pair_sim_off[k] + n * m].reshape(n, m)
                assert np.array_equal(got.view(np.uint64), ref.view(np.uint64)), key
                want = [(float.fromhex(s), i, j) for s, i, j in fx[key]["indices"]]
                assert [(float(r["score"]), int(r["i"]), int(r["j"])) for r in per_pair[k]] == want, key
