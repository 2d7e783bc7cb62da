"""Randomised parity: the CUDA path against the C oracle on generated batches.

hypothesis draws small vocabularies (many repeated and shared tokens),
pairs on both sides of the 64-sentence tile boundary, target documents
with more distinct tokens than one shared-memory chunk, sentences up to 300
tokens (past the 255-token limit of pair_kernel), dictionaries with
duplicate and zero-probability entries and tokens without any row,
probabilities of every float class (subnormal, > 1, NaN, overflowing, inf), and
random mining settings, sent in the int32 or the compact wire form.  Score
matrices must be bit-identical, and match counts and mined (score, i, j)
triples equal.
"""

import numpy as np
import pytest

hypothesis = pytest.importorskip("hypothesis")
from hypothesis import HealthCheck, given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402

import helpers as H  # noqa: E402
import oracle  # noqa: E402

pytestmark = pytest.mark.gpu


@st.composite
def batches(draw):
    from paper_1512_01641_b200.packing import PackedBatch, unique_counts

    uniform = draw(st.booleans())  # uniform ids over a large vocabulary: > 1024 distinct targets (chunking)
    vocab = draw(st.integers(2000, 6000)) if uniform else draw(st.integers(4, 400))
    n_pairs = draw(st.integers(1, 4))
    rng = np.random.default_rng(draw(st.integers(0, 2**32 - 1)))
    long_sentences = draw(st.booleans())
    sizes = [(int(rng.integers(1, 71)), int(rng.integers(1, 71))) for _ in range(n_pairs)]
    sent_len, pair_src, pair_tgt = [], [], []
    for n, m in sizes:
        pair_src.append(len(sent_len))
        sent_len += list(rng.integers(1, 40, size=n))
        pair_tgt.append(len(sent_len))
        sent_len += list(rng.integers(1, 40, size=m))
    sent_len = np.array(sent_len, dtype=np.int32)
    if long_sentences:
        k = rng.integers(0, sent_len.size)
        sent_len[k] = int(rng.integers(200, 301))
    T = int(sent_len.sum())
    tokens = rng.integers(0, vocab, size=T) if uniform else rng.zipf(1.3, size=T) % vocab
    off = np.zeros(sent_len.size, dtype=np.int64)
    np.cumsum(sent_len[:-1], out=off[1:])
    n = np.array([a for a, _ in sizes], dtype=np.int32)
    m = np.array([b for _, b in sizes], dtype=np.int32)
    sim_off = np.zeros(n_pairs, dtype=np.int64)
    np.cumsum((n.astype(np.int64) * m)[:-1], out=sim_off[1:])
    batch = PackedBatch(
        tokens=tokens.astype(np.int32), sent_tok_off=off, sent_len=sent_len,
        sent_uniq=unique_counts(tokens.astype(np.int32), sent_len).astype(np.int32),
        sent_chars=(sent_len * rng.integers(2, 9, size=sent_len.size)).astype(np.int32),
        pair_src=np.array(pair_src, dtype=np.int64), pair_n=n, pair_tgt=np.array(pair_tgt, dtype=np.int64),
        pair_m=m, pair_sim_off=sim_off)
    n_entries = int(rng.integers(0, 6 * vocab))
    src = rng.integers(0, vocab, size=n_entries).astype(np.int32)
    tgt = rng.integers(0, vocab, size=n_entries).astype(np.int32)
    prob = np.round(rng.random(n_entries), 6)
    prob[rng.random(n_entries) < 0.05] = 0.0  # dropped like read_lexicon + the p > 0 rule
    extreme = draw(st.sampled_from([None, None, "fine", "huge", "inf"]))
    if extreme:  # every float class read_lexicon admits (tests/helpers.py)
        prob = H.extreme_probabilities(prob, extreme, seed=int(rng.integers(0, 2**31)))
    gap = draw(st.sampled_from([0.0, 0.5, 1.3, 2.0, 3.7]))
    thr = draw(st.sampled_from([0.0, 0.3, 0.5, 0.9, 1.0]))
    wire = draw(st.booleans())  # bimine_mine_host's compact wire form (24-bit ids, uint16 sentence arrays)
    return batch, (src, tgt, prob), gap, thr, wire


@settings(max_examples=60, deadline=None, derandomize=True, suppress_health_check=list(HealthCheck))
@given(batches())
def test_random_batches_match_oracle(case):
    from paper_1512_01641_b200 import engine as E
    from paper_1512_01641_b200.classifier import model_vector

    batch, (src, tgt, prob), gap, thr, wire = case
    model = model_vector(H.synth_model())
    od = oracle.OracleDict(src, tgt, prob)
    want_sim = oracle.score_batch(od, model, batch)
    want_counts, want_rows = oracle.mine_batch(od, model, batch, gap=gap, threshold=thr)
    dd = E.LexiconContext(vocab=None, coo=(src, tgt, prob), devices={}).on(E.current_device())
    sent = batch.with_24bit_tokens().with_narrow_sentences() if wire else batch
    counts, matches, sim = E.mine_host(dd, model, sent, gap, thr, -1.0, 1.0, want_sim=True)
    assert np.array_equal(sim.view(np.uint64), want_sim.view(np.uint64))
    assert np.array_equal(counts, want_counts)
    flat = np.concatenate(want_rows) if want_rows else np.zeros(0, dtype=matches.dtype)
    assert np.array_equal(matches.view(np.uint8), flat.view(np.uint8))


@st.composite
def nw_problems(draw):
    rng = np.random.default_rng(draw(st.integers(0, 2**32 - 1)))
    n, m = draw(st.integers(1, 300)), draw(st.integers(1, 300))
    kind = draw(st.sampled_from(["uniform", "binary", "levels"]))
    if kind == "uniform":
        sim = rng.random((n, m))
    elif kind == "binary":
        sim = (rng.random((n, m)) > 0.7).astype(np.float64)
    else:  # few distinct values: tie-heavy DP
        sim = rng.integers(0, 4, size=(n, m)) / 3.0
    gap = draw(st.sampled_from([0.0, 0.25, 0.5, 1.0, 2.0]))
    return sim, gap


@settings(max_examples=40, deadline=None, derandomize=True, suppress_health_check=list(HealthCheck))
@given(st.lists(nw_problems(), min_size=1, max_size=3))
def test_random_nw_problems_match_oracle(problems):
    """Small (warp per problem) and large (cluster band pipeline) NW paths,
    one batch: step codes and dp[N][M] bit-identical to the oracle."""
    from paper_1512_01641_b200 import engine as E

    sims = [s for s, _ in problems]
    gaps = [g for _, g in problems]
    out = E.nw_steps_host(sims, gaps, -1.0, 1.0)
    for (sim, gap), (codes, score) in zip(problems, out):
        want, _, _, want_score = oracle.nw_align(sim, -1.0, 1.0, gap)
        assert np.array_equal(codes, want)
        assert np.array_equal(np.array([score]).view(np.uint64), np.array([want_score]).view(np.uint64))
