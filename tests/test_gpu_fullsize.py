"""Parity at BASELINE.json's full sizes.

* C2 (10k pairs ~50x50, 1M-entry dictionary): score matrices and mined
  triples of the whole batch, bit-exact against the C oracle.
* C3 (one 4096x4096 pair): NW + traceback + filter in full against the
  oracle run on the GPU's score matrix; 48 sampled rows of the score matrix
  against the oracle.  A cell depends only on its two sentences
  (classifier.py:62-97), so a sub-pair made of those rows scores identically.
* C4 (1k pairs x 64 (threshold, gap) trials): per (pair, trial) match counts
  and agreement against the oracle.
* C5's total (1M pairs, 2.5G cells: flat offsets past 2^31) on one GPU: C2's
  pairs repeated 100 times over the same sentences.  Every replica's counts
  and triples equal the first copy's; the C2 test pins that copy to the
  oracle.
"""

import numpy as np
import pytest

import helpers as H

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU containers
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
from paper_1512_01641_b200 import engine as E  # noqa: E402
from paper_1512_01641_b200 import synth  # noqa: E402
from paper_1512_01641_b200.classifier import model_vector  # noqa: E402
from paper_1512_01641_b200.packing import PackedBatch  # noqa: E402

GAP, THRESHOLD, MISMATCH, BONUS = 2.0, 0.5, -1.0, 1.0  # MiningConfig defaults (align.py:78-82)


def bits_equal(a, b):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


@pytest.fixture(scope="module", autouse=True)
def _oracle():
    oracle.build()


def _device_dict(corpus):
    d = corpus.dictionary
    return E.LexiconContext(vocab=None, coo=(d.src, d.tgt, d.prob), devices={}).on(E.current_device())


@pytest.fixture(scope="module")
def c2():
    corpus = synth.make_config(2)
    assert corpus.batch.n_pairs == 10_000
    return corpus


def test_c2_full_batch_bit_exact(c2):
    model = model_vector(H.synth_model())
    d = c2.dictionary
    od = oracle.OracleDict(d.src, d.tgt, d.prob)
    batch = c2.batch
    counts, matches, sim = E.mine_host(_device_dict(c2), model, batch, GAP, THRESHOLD, MISMATCH, BONUS,
                                       want_sim=True)
    assert bits_equal(sim, oracle.score_batch(od, model, batch))
    want_counts, want_rows = oracle.mine_batch(od, model, batch, GAP, THRESHOLD, MISMATCH, BONUS)
    assert np.array_equal(counts, want_counts)
    assert np.array_equal(matches.view(np.uint8), np.concatenate(want_rows).view(np.uint8))
    assert int(counts.sum()) > 100_000  # the workload mines (not a vacuous comparison)


def _rows_subpair(batch, rows):
    """One pair: source sentences `rows` of pair 0, all its target sentences."""
    src = batch.pair_src[0] + np.asarray(rows, dtype=np.int64)
    tgt = batch.pair_tgt[0] + np.arange(batch.pair_m[0], dtype=np.int64)
    sent = np.concatenate([src, tgt])
    tok = np.concatenate([batch.tokens[batch.sent_tok_off[s]: batch.sent_tok_off[s] + batch.sent_len[s]]
                          for s in sent.tolist()])
    return PackedBatch.from_token_lengths(
        tok, batch.sent_len[sent], batch.sent_chars[sent],
        np.array([0], np.int64), np.array([len(rows)], np.int32),
        np.array([len(rows)], np.int64), np.array([batch.pair_m[0]], np.int32),
        sent_uniq=batch.sent_uniq[sent])


def test_c3_full_pair():
    corpus = synth.make_config(3)
    batch = corpus.batch
    n, m = int(batch.pair_n[0]), int(batch.pair_m[0])
    assert (n, m) == (4096, 4096)
    model = model_vector(H.synth_model())
    d = corpus.dictionary
    od = oracle.OracleDict(d.src, d.tgt, d.prob)
    counts, matches, sim = E.mine_host(_device_dict(corpus), model, batch, GAP, THRESHOLD, MISMATCH, BONUS,
                                       want_sim=True)
    sim = sim.reshape(n, m)
    rows = np.sort(np.random.default_rng(3).choice(n, size=48, replace=False))
    rows[0], rows[-1] = 0, n - 1  # both edges of the first and last 64x64 tile rows
    want_rows = oracle.score_batch(od, model, _rows_subpair(batch, rows)).reshape(len(rows), m)
    assert bits_equal(sim[rows], want_rows)
    # NW + traceback + filter of the whole 4096x4096 matrix
    codes, si, sj, _ = oracle.nw_align(sim, MISMATCH, BONUS, GAP)
    keep = (codes == 0) & (sim[si, sj] >= THRESHOLD)
    assert counts[0] == int(keep.sum()) > 1000
    assert np.array_equal(matches["i"], si[keep]) and np.array_equal(matches["j"], sj[keep])
    assert bits_equal(matches["score"], sim[si[keep], sj[keep]])


def test_c4_full_tuning_sweep():
    from paper_1512_01641_b200 import align as A
    from paper_1512_01641_b200 import tuning as T

    corpus = synth.make_config(4)
    batch = corpus.batch
    P = batch.n_pairs
    assert P == 1000
    thr, gaps = T.draw_trials(A.MiningConfig(), 64, 7)
    model = model_vector(H.synth_model())
    refs = [list(map(tuple, corpus.reference[p])) for p in range(P)]
    counts, matched = E.tune_device(_device_dict(corpus), model, batch, thr, gaps, MISMATCH, BONUS, refs)
    counts = np.asarray(counts).reshape(P, 64)
    matched = np.asarray(matched).reshape(P, 64)
    d = corpus.dictionary
    sims = oracle.score_batch(oracle.OracleDict(d.src, d.tgt, d.prob), model, batch)
    for p in range(P):
        n, m = int(batch.pair_n[p]), int(batch.pair_m[p])
        sim = sims[batch.pair_sim_off[p]: batch.pair_sim_off[p] + n * m].reshape(n, m)
        ref = refs[p]
        for t in range(64):
            codes, si, sj, _ = oracle.nw_align(sim, MISMATCH, BONUS, gaps[t])
            keep = (codes == 0) & (sim[si, sj] >= thr[t])
            cand = list(zip(si[keep].tolist(), sj[keep].tolist()))
            assert counts[p, t] == len(cand), (p, t)
            want = 0
            if ref and cand:  # alignment_agreement's NW (tuning.py:60-82)
                eq = np.array([[1.0 if a == b else 0.0 for b in ref] for a in cand])
                ec, ei, ej, _ = oracle.nw_align(eq, -1.0, 1.0, 1.0)
                want = int(((ec == 0) & (eq[ei, ej] == 1.0)).sum())
            assert matched[p, t] == want, (p, t)
    assert matched.sum() > 0


def test_c5_total_size_by_replication(c2):
    """1M pairs / 2.54G cells on one GPU: replicas of C2's pairs (sharing its
    sentences) mine exactly like the first copy."""
    R = 100
    b = c2.batch
    P = b.n_pairs
    pn, pm = np.tile(b.pair_n, R), np.tile(b.pair_m, R)
    cells = pn.astype(np.int64) * pm
    sim_off = np.zeros(P * R, dtype=np.int64)
    np.cumsum(cells[:-1], out=sim_off[1:])
    assert int(sim_off[-1] + cells[-1]) > 2**31
    big = PackedBatch(tokens=b.tokens, sent_tok_off=b.sent_tok_off, sent_len=b.sent_len, sent_uniq=b.sent_uniq,
                      sent_chars=b.sent_chars, pair_src=np.tile(b.pair_src, R), pair_n=pn,
                      pair_tgt=np.tile(b.pair_tgt, R), pair_m=pm, pair_sim_off=sim_off)
    model = model_vector(H.synth_model())
    dd = _device_dict(c2)
    counts, matches, _ = E.mine_host(dd, model, big, GAP, THRESHOLD, MISMATCH, BONUS)
    counts = counts.copy()
    matches = matches.copy()
    c1, m1, _ = E.mine_host(dd, model, b, GAP, THRESHOLD, MISMATCH, BONUS)
    assert np.array_equal(counts, np.tile(c1, R))
    per = int(c1.sum())
    assert matches.shape[0] == R * per
    first = m1.view(np.uint8).reshape(per, -1)
    allm = matches.view(np.uint8).reshape(R, per, -1)
    for r in range(R):
        assert np.array_equal(allm[r], first), r
    torch.cuda.empty_cache()
