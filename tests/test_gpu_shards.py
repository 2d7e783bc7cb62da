"""Sharded and oversized batches on the device.

* mine_corpus's threaded path: the input cut into several chunks that go
  round-robin to the visible GPUs (all to cuda:0 on a one-GPU box); rows are
  identical for any worker count and chunk size, and equal to the C oracle's
  triples rendered as sentence text.
* A document a device limit rejects (a sentence of more than 16384 tokens)
  is reported as that pair's failure; the other pairs mine exactly as
  without it (the reference never raises per pair, align.py:405-447).
* More than 65,535 pairs with one pair larger than 64x64 in one call: the
  small pairs keep the one-warp NW, the large one goes to the cluster
  kernel.
* One device batch with more than 2^31 tokens (C5's 2.2G tokens on one
  GPU): flat token offsets past int32.
"""

import numpy as np
import pytest

import helpers as H

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU containers
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
from paper_1512_01641_b200 import align as A  # noqa: E402
from paper_1512_01641_b200 import engine as E  # noqa: E402
from paper_1512_01641_b200 import synth  # noqa: E402
from paper_1512_01641_b200.classifier import model_vector  # noqa: E402
from paper_1512_01641_b200.corpus import Document, DocumentPair  # noqa: E402
from paper_1512_01641_b200.lexicon import Lexicon  # noqa: E402
from paper_1512_01641_b200.packing import PackedBatch  # noqa: E402

GAP, THRESHOLD, MISMATCH, BONUS = 2.0, 0.5, -1.0, 1.0


@pytest.fixture(scope="module", autouse=True)
def _oracle():
    oracle.build()


@pytest.fixture(scope="module")
def docs():
    corpus = synth.make_config(2, n_pairs=160)
    pairs = []
    for p in range(corpus.batch.n_pairs):
        src, tgt = corpus.pair_sentences(p)
        pairs.append(DocumentPair(f"t{p}", Document(f"s{p}", "pl", str(p), tuple(src)),
                                  Document(f"d{p}", "en", str(p), tuple(tgt))))
    return corpus, pairs, Lexicon(corpus.dictionary.table())


def _oracle_rows(corpus, pairs):
    """The C oracle's mined triples of the corpus, as (score, src, tgt) text rows."""
    d = corpus.dictionary
    model = model_vector(H.synth_model())
    _, per_pair = oracle.mine_batch(oracle.OracleDict(d.src, d.tgt, d.prob), model, corpus.batch,
                                    GAP, THRESHOLD, MISMATCH, BONUS)
    rows = []
    for p, r in zip(pairs, per_pair):
        rows.extend((float(x["score"]), p.source.sentences[int(x["i"])], p.target.sentences[int(x["j"])]) for x in r)
    return rows


@pytest.mark.parametrize("workers,chunk", [(1, 16384), (2, 16384), (3, 50), (7, 23)])
def test_mine_corpus_shards_round_robin_bit_exact(docs, monkeypatch, workers, chunk):
    corpus, pairs, lex = docs
    monkeypatch.setattr(A, "CHUNK_PAIRS", chunk)
    out = A.mine_corpus(H.synth_model(), lex, pairs, A.MiningConfig(workers=workers))
    assert out.failures == ()
    assert len(A._chunk_bounds(len(pairs), workers)) >= min(workers, len(pairs))
    want = _oracle_rows(corpus, pairs)
    assert len(out.rows) == len(want) > 100
    for got, w in zip(out.rows, want):
        assert got[1:] == w[1:] and np.float64(got[0]).view(np.uint64) == np.float64(w[0]).view(np.uint64)


def test_mine_corpus_device_limit_failure_isolated(docs):
    corpus, pairs, lex = docs
    words = corpus.dictionary.words(np.arange(20_000) % 1000)
    huge = " ".join(words) + "."  # one sentence of 20,000 tokens: past the device's 16384
    bad = DocumentPair("huge", Document("hs", "pl", "h", (huge,) + pairs[1].source.sentences),
                       Document("ht", "en", "h", pairs[1].target.sentences))
    mixed = [pairs[0], bad, pairs[2]]
    out = A.mine_corpus(H.synth_model(), lex, mixed, A.MiningConfig())
    assert [f[0] for f in out.failures] == ["huge"]
    assert out.failures[0][1].startswith("pair huge: ")
    clean = A.mine_corpus(H.synth_model(), lex, [pairs[0], pairs[2]], A.MiningConfig())
    assert out.rows == clean.rows and len(clean.rows) > 0


def _replicate(batch, reps, extra=None):
    """`reps` copies of the batch's pairs over its sentences (+ optional
    extra pair descriptors appended)."""
    pn, pm = np.tile(batch.pair_n, reps), np.tile(batch.pair_m, reps)
    ps, pt = np.tile(batch.pair_src, reps), np.tile(batch.pair_tgt, reps)
    if extra is not None:
        pn, pm = np.append(pn, extra[1]), np.append(pm, extra[3])
        ps, pt = np.append(ps, extra[0]), np.append(pt, extra[2])
    cells = pn.astype(np.int64) * pm
    off = np.zeros(pn.shape[0], dtype=np.int64)
    np.cumsum(cells[:-1], out=off[1:])
    return PackedBatch(tokens=batch.tokens, sent_tok_off=batch.sent_tok_off, sent_len=batch.sent_len,
                       sent_uniq=batch.sent_uniq, sent_chars=batch.sent_chars, pair_src=ps, pair_n=pn,
                       pair_tgt=pt, pair_m=pm, pair_sim_off=off)


def _dd(corpus):
    d = corpus.dictionary
    return E.LexiconContext(vocab=None, coo=(d.src, d.tgt, d.prob), devices={}).on(E.current_device())


def test_more_than_65535_pairs_with_one_large_pair():
    small = synth.make_config(2, n_pairs=1000)
    big = synth.make_corpus(20261018 + 1003, 1, 200_000, (70, 65), dictionary=small.dictionary)
    # one batch: the small pairs' sentences, then the large pair's
    b, g = small.batch, big.batch
    S0, T0 = b.n_sentences, b.n_tokens
    merged = PackedBatch.from_token_lengths(
        np.concatenate([b.tokens, g.tokens]), np.concatenate([b.sent_len, g.sent_len]),
        np.concatenate([b.sent_chars, g.sent_chars]), b.pair_src, b.pair_n, b.pair_tgt, b.pair_m,
        sent_uniq=np.concatenate([b.sent_uniq, g.sent_uniq]))
    reps = 70  # 70,000 small pairs
    batch = _replicate(merged, reps, extra=(S0 + g.pair_src[0], g.pair_n[0], S0 + g.pair_tgt[0], g.pair_m[0]))
    assert batch.n_pairs > 65_535 and int(batch.pair_n.max()) > 64
    model = model_vector(H.synth_model())
    counts, matches, _ = E.mine_host(_dd(small), model, batch, GAP, THRESHOLD, MISMATCH, BONUS)
    counts, matches = counts.copy(), matches.copy()
    d = small.dictionary
    od = oracle.OracleDict(d.src, d.tgt, d.prob)
    wc, wr = oracle.mine_batch(od, model, b, GAP, THRESHOLD, MISMATCH, BONUS)
    gc, gr = oracle.mine_batch(od, model, g, GAP, THRESHOLD, MISMATCH, BONUS)
    assert np.array_equal(counts, np.concatenate([np.tile(wc, reps), gc]))
    per = int(wc.sum())
    first = np.concatenate(wr).view(np.uint8)
    got = matches.view(np.uint8).reshape(-1, 16)
    for r in range(reps):
        assert np.array_equal(got[r * per:(r + 1) * per].ravel(), first), r
    assert np.array_equal(got[reps * per:].ravel(), np.concatenate(gr).view(np.uint8))
    assert S0 + T0 > 0


def test_single_device_more_than_2e31_tokens():
    """C5's token volume on one GPU: 100 token copies of C2 (distinct
    storage, so sentence offsets run past 2^31); every copy mines like the
    first, which test_gpu_fullsize pins to the oracle."""
    c2 = synth.make_config(2)
    b = c2.batch
    R = 100
    T, S = b.n_tokens, b.n_sentences
    assert T * R > 2**31
    tokens = np.tile(b.tokens, R)
    sent_len = np.tile(b.sent_len, R)
    big = PackedBatch.from_token_lengths(
        tokens, sent_len, np.tile(b.sent_chars, R),
        (b.pair_src[None, :] + S * np.arange(R)[:, None]).ravel(), np.tile(b.pair_n, R),
        (b.pair_tgt[None, :] + S * np.arange(R)[:, None]).ravel(), np.tile(b.pair_m, R),
        sent_uniq=np.tile(b.sent_uniq, R))
    del tokens
    assert int(big.sent_tok_off[-1]) > 2**31
    model = model_vector(H.synth_model())
    dd = _dd(c2)
    counts, matches, _ = E.mine_host(dd, model, big, GAP, THRESHOLD, MISMATCH, BONUS)
    counts, matches = counts.copy(), matches.copy()
    c1, m1, _ = E.mine_host(dd, model, b, GAP, THRESHOLD, MISMATCH, BONUS)
    assert np.array_equal(counts, np.tile(c1, R))
    per = int(c1.sum())
    first = m1.view(np.uint8).reshape(per, -1)
    allm = matches.view(np.uint8).reshape(R, per, -1)
    for r in range(R):
        assert np.array_equal(allm[r], first), r
    del big, matches
    torch.cuda.empty_cache()


def test_agreement_beyond_shared_memory_cap():
    """alignment_agreement (tuning.py:60-82) on device for lists whose
    direction table exceeds shared memory (500 candidates x 400 references:
    ~221 KB per warp): the global-scratch path, against the oracle's NW on
    the 0/1 equality matrix."""
    from paper_1512_01641_b200 import _native as N

    rng = np.random.default_rng(11)
    P, S = 3, 2
    K, R = 500, 400
    dev = "cuda:0"
    cand_lists, ref_lists = [], []
    for p in range(P * S):
        ii = np.sort(rng.choice(900, K, replace=False))
        jj = np.sort(rng.choice(900, K, replace=False))
        cand_lists.append(list(zip(ii.tolist(), jj.tolist())))
    for p in range(P):
        base = cand_lists[p * S]
        keep = sorted(rng.choice(K, 250, replace=False).tolist())
        extra = [(int(a), int(b)) for a, b in zip(rng.integers(0, 900, R - 250), rng.integers(0, 900, R - 250))]
        ref_lists.append(sorted([base[k] for k in keep] + extra))
    slots = np.zeros(P * S * K, dtype=N.MATCH_DTYPE)
    for q, lst in enumerate(cand_lists):
        slots["i"][q * K:(q + 1) * K] = [a for a, _ in lst]
        slots["j"][q * K:(q + 1) * K] = [b for _, b in lst]
    out_off = np.arange(P * S, dtype=np.int64) * K
    counts = np.full(P * S, K, dtype=np.int32)
    ref_ij = np.array([x for r in ref_lists for pr in r for x in pr], dtype=np.int32)
    ref_off = np.arange(P, dtype=np.int64) * R
    ref_len = np.full(P, R, dtype=np.int32)
    t = {k: torch.from_numpy(v).to(dev) for k, v in dict(slots=slots.view(np.uint8), out_off=out_off, counts=counts,
                                                         ref_ij=ref_ij, ref_off=ref_off, ref_len=ref_len).items()}
    matched = torch.empty(P * S, dtype=torch.int32, device=dev)
    L = N.load()
    N.check(L.bimine_agreement_batch(t["slots"].data_ptr(), t["out_off"].data_ptr(), t["counts"].data_ptr(), P, S,
                                     t["ref_ij"].data_ptr(), t["ref_off"].data_ptr(), t["ref_len"].data_ptr(), K, R,
                                     matched.data_ptr(), E.stream_ptr()))
    got = matched.cpu().numpy()
    for q in range(P * S):
        cand, ref = cand_lists[q], ref_lists[q // S]
        eq = np.array([[1.0 if a == b else 0.0 for b in ref] for a in cand])
        codes, si, sj, _ = oracle.nw_align(eq, -1.0, 1.0, 1.0)
        want = int(((codes == 0) & (eq[si, sj] == 1.0)).sum())
        assert got[q] == want, (q, got[q], want)
        if q % S == 0:  # the setting whose candidates the references were drawn from
            assert want > 100


def test_24bit_token_ids_mine_identically():
    """bimine_mine_host and the device-resident score path read 24-bit
    packed ids (the compact upload form) with the same results as int32,
    including ids at the 8/16/24-bit boundaries (a remapped vocabulary)."""
    c = synth.make_config(2, n_pairs=300)
    b = c.batch
    model = model_vector(H.synth_model())
    dd = _dd(c)
    c32, m32, s32 = E.mine_host(dd, model, b, GAP, THRESHOLD, MISMATCH, BONUS, want_sim=True)
    c32, m32, s32 = c32.copy(), m32.copy(), s32.copy()
    p = b.with_24bit_tokens()
    c24, m24, s24 = E.mine_host(dd, model, p, GAP, THRESHOLD, MISMATCH, BONUS, want_sim=True)
    assert np.array_equal(c24, c32) and np.array_equal(m24.view(np.uint8), m32.view(np.uint8))
    assert np.array_equal(s24.view(np.uint64), s32.view(np.uint64))
    sim = torch.empty(b.n_cells, dtype=torch.float64, device="cuda:0")
    E.score_device(dd, model, E.DeviceBatch(p, 0), sim)
    assert np.array_equal(sim.cpu().numpy().view(np.uint64), s32.view(np.uint64))
    # ids near 2^24: a bijective remap of every id used (dictionary included) keeps the scores
    d = c.dictionary
    used = np.unique(np.concatenate([b.tokens, d.src, d.tgt]))
    hi = (1 << 24) - 1 - np.arange(used.size, dtype=np.int64)
    hi[: min(3, hi.size)] = [0, 255, 256][: min(3, hi.size)]
    remap = dict(zip(used.tolist(), hi.tolist()))
    f = np.vectorize(remap.__getitem__, otypes=[np.int32])
    rb = PackedBatch(**{**{k: getattr(b, k) for k in ("sent_tok_off", "sent_len", "sent_uniq", "sent_chars",
                                                        "pair_src", "pair_n", "pair_tgt", "pair_m", "pair_sim_off")},
                        "tokens": f(b.tokens)})
    rdd = E.LexiconContext(vocab=None, coo=(f(d.src), f(d.tgt), d.prob), devices={}).on(0)
    cr, mr, sr = E.mine_host(rdd, model, rb.with_24bit_tokens(), GAP, THRESHOLD, MISMATCH, BONUS, want_sim=True)
    assert np.array_equal(sr.view(np.uint64), s32.view(np.uint64)) and np.array_equal(cr, c32)
