"""GPU parity: the CUDA path against the reference's fixtures and the oracle.

Bit-exact everywhere: score matrices (binary64 bit patterns), alignment
step lists, Alignment.score, mined (score, i, j) triples.  The north-star
tolerance for scores is 1e-6 relative; the kernels meet it with zero
error, and the tests hold them to that.
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

SCORE_RTOL = 1e-6  # BASELINE.json north_star tolerance for scores


def bits_equal(a, b):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


@pytest.fixture(scope="module", autouse=True)
def _oracle():
    oracle.build()


def test_native_library_is_loaded():
    from paper_1512_01641_b200 import _native

    L = _native.load()
    assert b"sm_100a" in L.bimine_version()


# ---------------------------------------------------------------- exp

def test_device_exp_matches_reference_math_exp():
    z = H.load_npz("exp_golden.npz")
    assert bits_equal(E.exp_device(z["x"]), z["y"])


def test_device_exp_matches_host_libm_randomised():
    rng = np.random.default_rng(7)
    x = np.concatenate([-rng.uniform(0, 700, 4_000_000), rng.uniform(-745, 710, 2_000_000),
                        rng.uniform(-1, 1, 1_000_000), -rng.uniform(511.5, 512.5, 500_000)])
    assert bits_equal(E.exp_device(x), oracle.exp_array(x))


# ---------------------------------------------------------------- NW

@pytest.mark.parametrize("family", H.NW_FAMILIES)
def test_nw_reference_families(family):
    sims = list(H.nw_family_sims(family))
    fx = H.nw_family(family)
    gaps = [float(g) for _, _, _, g in fx]
    out = E.nw_steps_host(sims, gaps, H.NW_MISMATCH, H.NW_BONUS)
    for (codes, score), (want, want_score, shape, _) in zip(out, fx):
        assert np.array_equal(codes, want)
        assert score == want_score


def test_nw_align_api_and_demo_fixtures():
    # demos.py:18-29 / test_align.py:221-251
    def exact(src, tgt):
        return np.array([[1.0 if s == t else 0.0 for t in tgt] for s in src])

    demo = A.MiningConfig(threshold=0.5, gap_penalty=5.0, match_bonus=9.0, mismatch_cost=-4.0)
    src, tgt = ("a", "d", "c", "d", "e"), ("a", "d", "e", "g", "f")
    al = A.nw_align(exact(src, tgt), demo)
    sl, tl = [], []
    for s in al.steps:
        if isinstance(s, A.Match):
            sl.append(src[s.i]); tl.append(tgt[s.j])
        elif isinstance(s, A.GapSource):
            sl.append(src[s.i]); tl.append("-")
        else:
            sl.append("-"); tl.append(tgt[s.j])
    assert ", ".join(tl) == "a, d, -, -, e, g, f"
    assert ", ".join(sl) == "a, d, c, d, e, -, -"
    ws, wt = ("tablets", "make", "people", "spoil", "children"), ("tablets", "make", "children", "very", "addicted")
    al = A.nw_align(exact(ws, wt), demo)
    assert {(ws[s.i], wt[s.j]) for s in al.steps if isinstance(s, A.Match)} == {
        ("tablets", "tablets"), ("make", "make"), ("children", "children")}
    eye = A.nw_align(np.eye(5), A.MiningConfig(gap_penalty=1.0))
    assert eye.steps == tuple(A.Match(i, i) for i in range(5)) and eye.score == 5.0
    assert A.nw_align_wavefront(np.eye(5), A.MiningConfig(gap_penalty=1.0), 4) == eye
    with pytest.raises(ValueError):
        A.nw_align(np.zeros((0, 3)), A.MiningConfig())
    with pytest.raises(ValueError):
        A.nw_align(np.array([[0.5, 1.5]]), A.MiningConfig())
    with pytest.raises(ValueError):
        A.nw_align(np.array([[np.nan]]), A.MiningConfig())
    with pytest.raises(ValueError):
        A.nw_align_wavefront(np.eye(2), A.MiningConfig(), 0)


@pytest.mark.parametrize("shape", [(1, 1), (1, 70), (70, 1), (31, 33), (32, 32), (33, 31), (64, 65), (200, 220), (513, 300)])
def test_nw_steps_match_oracle_random(shape):
    rng = np.random.default_rng(sum(shape))
    sims = [rng.random(shape) for _ in range(3)] + [rng.integers(0, 2, size=shape).astype(np.float64)]
    gaps = [0.0, 0.7, 2.0, 0.5]
    out = E.nw_steps_host(sims, gaps, -1.0, 1.0)
    for sim, g, (codes, score) in zip(sims, gaps, out):
        want, _, _, want_score = oracle.nw_align(sim, -1.0, 1.0, g)
        assert np.array_equal(codes, want)
        assert bits_equal(score, want_score)


def test_nw_fill_b1_contract_bit_identical():
    """bimine_nw_fill honours the reference FFI: caller boundaries, interior
    written in place, bit-identical to the reference fill (_nwcore.pyx:19-36)."""
    rng = np.random.default_rng(11)
    for shape in [(1, 1), (5, 4), (40, 33), (97, 130), (300, 64)]:
        sim = rng.random(shape)
        gap = float(rng.uniform(0, 3))
        want = oracle.nw_table(sim, -1.0, 1.0, gap)
        dp = np.empty_like(want)
        dp[0, :] = -gap * np.arange(shape[1] + 1, dtype=np.float64)
        dp[1:, 0] = -gap * np.arange(1, shape[0] + 1, dtype=np.float64)
        E.nw_fill_host(dp, sim, -1.0, 1.0, gap)
        assert bits_equal(dp, want)
        # arbitrary caller boundaries are used as given
        dp2 = np.zeros_like(want)
        dp2[0, :] = rng.normal(size=shape[1] + 1)
        dp2[1:, 0] = rng.normal(size=shape[0])
        ref = dp2.copy()
        oracle.lib().oracle_nw_fill(ref.ctypes.data_as(oracle._f64p), sim.ctypes.data_as(oracle._f64p),
                                    shape[0], shape[1], -1.0, 1.0, gap)
        E.nw_fill_host(dp2, sim, -1.0, 1.0, gap)
        assert bits_equal(dp2, ref)


# ---------------------------------------------------------------- score matrix

def test_toy_score_matrices_bit_exact():
    model, lex = H.toy_model(), H.toy_lexicon()
    for (src, tgt), ref in zip(H.toy_pairs(), H.toy_sims()):
        got = A.build_score_matrix(model, lex, src, tgt)
        assert bits_equal(got, ref)
        np.testing.assert_allclose(got, ref, rtol=SCORE_RTOL, atol=0)


def test_similarity_is_the_score_matrix_cell():
    """classifier.similarity (classifier.py:357-362) = the cell of the
    reference's score matrix, bit for bit; errors unprefixed."""
    from paper_1512_01641_b200.classifier import similarity

    model, lex = H.toy_model(), H.toy_lexicon()
    (src, tgt), ref = H.toy_pairs()[0], H.toy_sims()[0]
    for i in range(min(3, len(src))):
        for j in range(min(3, len(tgt))):
            assert bits_equal(np.array([similarity(model, src[i], tgt[j], lex)]), np.array([ref[i, j]]))
    with pytest.raises(ValueError, match=r"^untokenizable sentence: '\.\.\.'$"):
        similarity(model, "domo", "...", lex)


def test_extract_features_match_reference():
    """classifier.extract_features (features mode of the score kernel) =
    the reference's extract_features bit for bit (tests/golden/
    features_golden.json: every toy cell + edge pairs)."""
    from paper_1512_01641_b200.classifier import extract_features

    lex = H.toy_lexicon()
    for a, b, want in H.load_json("features_golden.json")["cells"]:
        got = extract_features(a, b, lex)
        assert [float(v).hex() for v in got] == want, (a, b)
    with pytest.raises(ValueError, match=r"^untokenizable sentence: '\.\.\.'$"):
        extract_features("...", "house", lex)


def test_score_matrix_errors_match_reference():
    model, lex = H.toy_model(), H.toy_lexicon()
    with pytest.raises(ValueError) as exc:
        A.build_score_matrix(model, lex, ["domo"], ["house", "..."])
    assert str(exc.value) == H.load_json("toy.json")["error_untokenizable"]
    with pytest.raises(ValueError):
        A.build_score_matrix(model, lex, [], ["house"])


@pytest.mark.parametrize("cfg", ["default", "strict", "loose"])
def test_toy_mining_rows_bit_exact(cfg):
    params = {
        "default": A.MiningConfig(),
        "strict": A.MiningConfig(threshold=0.8, gap_penalty=0.5),
        "loose": A.MiningConfig(threshold=0.0, gap_penalty=3.0, match_bonus=2.0, mismatch_cost=-0.5),
    }[cfg]
    model, lex = H.toy_model(), H.toy_lexicon()
    fx = H.load_json("toy.json")["pairs"]
    pairs = []
    for p in fx:
        pair = DocumentPair(
            topic_id=p["topic_id"],
            source=Document(id="s", lang="eo", title="t", sentences=tuple(p["source"])),
            target=Document(id="t", lang="en", title="t", sentences=tuple(p["target"])),
        )
        pairs.append(pair)
        rows = A.mine_document_pair(model, lex, pair, params, engine="nw")
        want = [(float.fromhex(s), a, b) for s, a, b in p[cfg]["rows"]]
        assert rows == want, p["topic_id"]
    outcome = A.mine_corpus(model, lex, pairs, params)
    assert outcome.failures == ()
    assert list(outcome.rows) == [(float.fromhex(s), a, b) for p in fx for s, a, b in p[cfg]["rows"]]


def test_mine_corpus_failures_and_order():
    model, lex = H.toy_model(), H.toy_lexicon()
    fx = H.load_json("toy.json")
    p0 = fx["pairs"][0]
    good = DocumentPair("alpha", Document("a", "eo", "t", tuple(p0["source"])), Document("b", "en", "t", tuple(p0["target"])))
    bad = DocumentPair("bad", Document("b1", "eo", "bad", ("...",)), Document("b2", "en", "bad", ("house",)))
    out = A.mine_corpus(model, lex, [good, bad], A.MiningConfig(), engine="nw")
    assert [list(f) for f in out.failures] == fx["mine_corpus_failures"]
    assert len(out.rows) > 0
    assert A.mine_corpus(model, lex, [], A.MiningConfig(workers=4)) == A.MiningOutcome((), ())
    with pytest.raises(ValueError, match="unknown engine"):
        A.mine_corpus(model, lex, [], A.MiningConfig(), engine="bogus")
    wide = A.mine_corpus(model, lex, [good, bad, good], A.MiningConfig(workers=16))
    narrow = A.mine_corpus(model, lex, [good, bad, good], A.MiningConfig(workers=1))
    assert wide == narrow


def _synth_check(corpus, pairs=None, threads=0):
    model = model_vector(H.synth_model())
    d = corpus.dictionary
    od = oracle.OracleDict(d.src, d.tgt, d.prob)
    batch = corpus.batch if pairs is None else corpus.batch.select(pairs)
    want_sim = oracle.score_batch(od, model, batch, threads)
    want_counts, want_rows = oracle.mine_batch(od, model, batch, threads=threads)
    ctx = E.LexiconContext(vocab=None, coo=(d.src, d.tgt, d.prob), devices={})
    dd = ctx.on(E.current_device())
    counts, matches, sim = E.mine_host(dd, model, batch, 2.0, 0.5, -1.0, 1.0, want_sim=True)
    assert bits_equal(sim, want_sim)
    assert np.array_equal(counts, want_counts)
    flat = np.concatenate(want_rows) if want_rows else np.zeros(0, dtype=matches.dtype)
    assert np.array_equal(matches.view(np.uint8), flat.view(np.uint8))
    return batch


def test_synthetic_fixtures_bit_exact():
    model = model_vector(H.synth_model())
    for name, corpus in [("synth_c1", synth.make_config(1)), ("synth_c2", synth.make_config(2, n_pairs=12))]:
        fx = H.load_json(f"{name}.json")
        sims = H.load_npz(f"{name}_sims.npz")
        d = corpus.dictionary
        ctx = E.LexiconContext(vocab=None, coo=(d.src, d.tgt, d.prob), devices={})
        dd = ctx.on(E.current_device())
        sub = corpus.batch.select(fx["pairs"])
        counts, matches, sim = E.mine_host(dd, model, sub, 2.0, 0.5, -1.0, 1.0, want_sim=True)
        pos = 0
        for k, p in enumerate(fx["pairs"]):
            ref = sims[f"sim{p}"]
            n, m = ref.shape
            assert bits_equal(sim[sub.pair_sim_off[k] : sub.pair_sim_off[k] + n * m].reshape(n, m), ref)
            want = [(float.fromhex(s), i, j) for s, i, j in fx["indices"][k]]
            got = [(float(r["score"]), int(r["i"]), int(r["j"])) for r in matches[pos : pos + counts[k]]]
            pos += counts[k]
            assert got == want


@pytest.mark.parametrize("wire", [False, True])
def test_extreme_probabilities_bit_exact(wire):
    """Dictionary probabilities of every float class (subnormal, tied, > 1,
    dropped zero/negative/NaN, sums overflowing to inf, +inf) through
    bimine_mine_host, int32 and compact wire form: score matrices and mined
    rows equal the reference's (extreme.json, made by make_golden.py)."""
    model = model_vector(H.synth_model())
    fx = H.load_json("extreme.json")
    sims = H.load_npz("extreme_sims.npz")
    for variant in H.EXTREME_VARIANTS:
        for cname, corpus, pairs in H.extreme_corpora():
            d = corpus.dictionary
            coo = (d.src, d.tgt, H.extreme_probabilities(d.prob, variant))
            dd = E.LexiconContext(vocab=None, coo=coo, devices={}).on(E.current_device())
            sub = corpus.batch.select(pairs)
            if wire:
                sub = sub.with_24bit_tokens().with_narrow_sentences()
            counts, matches, sim = E.mine_host(dd, model, sub, 2.0, 0.5, -1.0, 1.0, want_sim=True)
            pos = 0
            for k, p in enumerate(pairs):
                key = f"{variant}_{cname}_{p}"
                ref = sims[key]
                n, m = ref.shape
                assert bits_equal(sim[sub.pair_sim_off[k] : sub.pair_sim_off[k] + n * m].reshape(n, m), ref), key
                want = [(float.fromhex(s), i, j) for s, i, j in fx[key]["indices"]]
                got = [(float(r["score"]), int(r["i"]), int(r["j"])) for r in matches[pos : pos + counts[k]]]
                pos += counts[k]
                assert got == want, key


def test_synthetic_c2_batch_vs_oracle():
    _synth_check(synth.make_config(2, n_pairs=400))


def test_multi_tile_pairs_vs_oracle():
    """N, M > 64 (several CTAs per pair) and a C1-shaped pair."""
    corpus = synth.make_corpus(77, 6, 2_000, shape=(150, 131))
    _synth_check(corpus)
    _synth_check(synth.make_config(1))


def test_large_pair_global_scratch_vs_oracle():
    """A pair whose direction table does not fit shared memory."""
    corpus = synth.make_corpus(78, 1, 5_000, shape=(700, 650))
    _synth_check(corpus, threads=0)


def test_chunked_targets_and_long_sentences():
    """Sentences with many distinct tokens force several target chunks per
    tile; long sentences (> 64 tokens) exercise multi-segment streaming;
    repeated tokens exercise first-occurrence and multiplicity logic."""
    rng = np.random.default_rng(5)
    words = [f"w{k}" for k in range(3000)]
    trans = {w: {f"v{(k * 7 + j) % 3000}": float(round(rng.uniform(0.01, 1.0), 6)) for j in range(rng.integers(1, 9))}
             for k, w in enumerate(words[:2000])}
    # one long row (> inline candidate capacity) and a zero / negative entry
    trans["w1"] = {f"v{k}": 0.001 * (k + 1) for k in range(100)}  # longer than a segment
    trans["w2"]["v5"] = 0.0
    trans["w3"]["v6"] = -0.5
    lex = Lexicon(trans)

    def sent(n, side):
        pick = rng.integers(0, 3000, size=n)
        toks = [(words[i] if side == "s" else f"v{i}") for i in pick]
        if n > 3:
            toks[1] = toks[0]  # duplicates
            toks.append("zz")  # shared token on both sides
        return " ".join(toks) + "."

    pairs = [([sent(int(rng.integers(1, 150)), "s") for _ in range(70)],
              [sent(int(rng.integers(1, 150)), "t") for _ in range(90)]) for _ in range(2)]
    vocab, coo, batch = H.pack_pairs(lex, pairs)
    model = model_vector(H.toy_model())
    od = oracle.OracleDict(*coo)
    want = oracle.score_batch(od, model, batch)
    ctx = E.LexiconContext(vocab=vocab, coo=coo, devices={})
    got = E.score_host(ctx.on(E.current_device()), model, batch)
    assert bits_equal(got, want)
    for p, (src, tgt) in enumerate(pairs):
        g = A.build_score_matrix(H.toy_model(), lex, src, tgt)
        n, m = len(src), len(tgt)
        assert bits_equal(g, want[batch.pair_sim_off[p] : batch.pair_sim_off[p] + n * m].reshape(n, m))


def test_lexicon_duplicates_last_wins():
    """bimine_dict_create: repeated (src, tgt) keeps the last value."""
    src = np.array([0, 0, 0, 1], dtype=np.int32)
    tgt = np.array([5, 5, 6, 5], dtype=np.int32)
    prob = np.array([0.9, 0.2, 0.0, 0.4])
    d = E.DeviceDictionary(None, src, tgt, prob, E.current_device())
    assert d.n_entries == 2  # (0,5)=0.2, (1,5)=0.4; (0,6)=0 dropped


def test_sentences_longer_than_255_tokens_use_fallback_kernel():
    """u8 counters in pair_kernel: such pairs go to the tiled fallback; same bits."""
    rng = np.random.default_rng(8)
    lex = Lexicon({f"w{k}": {f"v{(k * 3 + j) % 500}": 0.1 + 0.1 * j for j in range(3)} for k in range(500)})
    def sent(n, pre):
        return " ".join(f"{pre}{i}" for i in rng.integers(0, 500, size=n)) + "."
    pairs = [([sent(300, "w"), sent(5, "w")], [sent(280, "v"), sent(4, "v"), sent(7, "v")]),
             ([sent(20, "w")] * 3, [sent(20, "v")] * 2)]
    vocab, coo, batch = H.pack_pairs(lex, pairs)
    model = model_vector(H.toy_model())
    want = oracle.score_batch(oracle.OracleDict(*coo), model, batch)
    ctx = E.LexiconContext(vocab=vocab, coo=coo, devices={})
    plan, _ = E.plan_batch(batch)
    assert plan.n_long == 1 and plan.n_tiles == 0
    got = E.score_host(ctx.on(E.current_device()), model, batch)
    assert bits_equal(got, want)
    # through bimine_mine_host too (it uploads sent_uniq only for such pairs)
    _, _, sim = E.mine_host(ctx.on(E.current_device()), model, batch, 2.0, 0.5, -1.0, 1.0, want_sim=True)
    assert bits_equal(sim, want)


def test_plan_tiles_for_large_pairs():
    corpus = synth.make_corpus(79, 3, 2_000, shape=(130, 65))
    plan, work = E.plan_batch(corpus.batch)
    assert plan.n_tiles == 3 * 3 * 2 and plan.n_long == 0
    assert work[: 3 * plan.n_tiles].reshape(-1, 3)[:, 0].tolist() == [0] * 6 + [1] * 6 + [2] * 6
    assert plan.n_large == 3 and work[3 * plan.n_tiles:3 * plan.n_tiles + 3].tolist() == [0, 1, 2]
    assert work[3 * plan.n_tiles + 3:].tolist() == [130, 65] * 3  # the large pairs' (N, M)
    _synth_check(corpus)


# ---------------------------------------------------------------- tuning (C4)

def test_tune_matches_reference_fixture():
    from paper_1512_01641_b200 import tuning as T

    fx = H.load_json("tune_golden.json")
    corpus = synth.make_config(fx["config"], n_pairs=fx["n_pairs"])
    lex = Lexicon(corpus.dictionary.table())
    samples = []
    for p in range(fx["n_pairs"]):
        src, tgt = corpus.pair_sentences(p)
        pair = DocumentPair(f"tune-{p}", Document(f"tune-{p}-s", "pl", str(p), tuple(src)),
                            Document(f"tune-{p}-t", "en", str(p), tuple(tgt)))
        samples.append(T.TuningSample(pair=pair, reference=tuple(tuple(r) for r in corpus.reference[p])))
    res = T.tune(H.synth_model(), lex, samples, budget=fx["budget"], seed=fx["seed"], engine="nw")
    want = fx["result"]
    assert res.threshold.hex() == want["threshold"] and res.gap_penalty.hex() == want["gap_penalty"]
    assert res.agreement.hex() == want["agreement"] and res.trials == want["trials"]
    assert [v.hex() for v in res.per_sample] == want["per_sample"]
    assert res.default_agreement.hex() == want["default_agreement"]


def test_alignment_agreement_kats():
    from paper_1512_01641_b200 import tuning as T

    assert T.alignment_agreement([(0, 0), (1, 1)], [(0, 0), (1, 1)]) == 100.0
    assert T.alignment_agreement([], [(0, 0)]) == 0.0
    assert T.alignment_agreement([], []) == 100.0
    assert T.alignment_agreement([(0, 0)], []) == 0.0
    assert T.alignment_agreement([(0, 0), (2, 2)], [(0, 0), (1, 1), (2, 2)]) == 200.0 / 3.0
    assert T.alignment_agreement([(0, 0), (1, 1), (2, 2)], [(0, 0), (2, 2)]) == 100.0
    for ref, cand, v in H.load_json("tune_golden.json")["agreement_kats"]:
        assert T.alignment_agreement([tuple(x) for x in cand], [tuple(x) for x in ref]).hex() == v


def test_tune_trials_agree_with_per_trial_recomputation():
    """Batched device agreements == per-trial mining + alignment_agreement."""
    from paper_1512_01641_b200 import tuning as T

    corpus = synth.make_config(4, n_pairs=5)
    lex = Lexicon(corpus.dictionary.table())
    model = H.synth_model()
    samples = []
    for p in range(5):
        src, tgt = corpus.pair_sentences(p)
        pair = DocumentPair(f"t{p}", Document("s", "pl", "t", tuple(src)), Document("t", "en", "t", tuple(tgt)))
        samples.append(T.TuningSample(pair=pair, reference=tuple(tuple(r) for r in corpus.reference[p])))
    res = T.tune(model, lex, samples, budget=12, seed=3)
    thr, gaps = T.draw_trials(A.MiningConfig(), 12, 3)
    rows = []
    for t in range(12):
        cfg = A.MiningConfig(threshold=thr[t], gap_penalty=gaps[t])
        row = []
        for s in samples:
            cand = [(i, j) for _, i, j in A.align_pair_indices(model, lex, s.pair, cfg)]
            row.append(T.alignment_agreement(cand, list(s.reference)))
        rows.append(row)
    want = T.select_best(np.array(rows), thr, gaps, 12)
    assert res == want


@pytest.mark.parametrize("layout", ["reversed_with_gaps", "one_gap"])
def test_mine_host_unpacked_sentence_offsets(layout):
    """bimine_mine_host rebuilds sent_tok_off from sent_len on the device
    unless the caller's offsets differ from that packed layout; then it uses
    the caller's.  Sentences stored out of order, with gaps, mine the same."""
    from paper_1512_01641_b200.packing import PackedBatch

    corpus = synth.make_config(2, n_pairs=40)
    d = corpus.dictionary
    model = model_vector(H.synth_model())
    dd = E.LexiconContext(vocab=None, coo=(d.src, d.tgt, d.prob), devices={}).on(E.current_device())
    b = corpus.batch
    want = E.mine_host(dd, model, b, 2.0, 0.5, -1.0, 1.0, want_sim=True)
    S = b.n_sentences
    order = np.arange(S)[::-1] if layout == "reversed_with_gaps" else np.arange(S)
    gap = 3 if layout == "reversed_with_gaps" else 0
    pieces, off, pos = [], np.zeros(S, dtype=np.int64), 0
    for s in order.tolist():
        if layout == "one_gap" and s == S // 2:
            pieces.append(np.full(5, 7, dtype=np.int32))
            pos += 5
        off[s] = pos
        pieces.append(b.tokens[b.sent_tok_off[s]: b.sent_tok_off[s] + b.sent_len[s]])
        pos += int(b.sent_len[s])
        if gap:
            pieces.append(np.full(gap, 123456, dtype=np.int32))
            pos += gap
    moved = PackedBatch(tokens=np.concatenate(pieces), sent_tok_off=off, sent_len=b.sent_len, sent_uniq=b.sent_uniq,
                        sent_chars=b.sent_chars, pair_src=b.pair_src, pair_n=b.pair_n, pair_tgt=b.pair_tgt,
                        pair_m=b.pair_m, pair_sim_off=b.pair_sim_off)
    got = E.mine_host(dd, model, moved, 2.0, 0.5, -1.0, 1.0, want_sim=True)
    assert np.array_equal(got[0], want[0])
    assert np.array_equal(got[1].view(np.uint8), want[1].view(np.uint8))
    assert bits_equal(got[2], want[2])


@pytest.mark.parametrize("fault", ["src_past_end", "tgt_negative", "empty_sentence", "tokens_past_end",
                                   "negative_sim_off"])
def test_mine_host_rejects_invalid_batches(fault):
    """bimine_mine_host launches the score kernel before it has validated
    the batch (each CTA bounds-checks its own pair): an invalid batch still
    gets the host's error, nothing is read or written out of range (the
    device stays usable), and the next valid call mines as before."""
    import dataclasses

    from paper_1512_01641_b200._native import BimineError

    corpus = synth.make_config(2, n_pairs=64)
    d = corpus.dictionary
    model = model_vector(H.synth_model())
    dd = E.LexiconContext(vocab=None, coo=(d.src, d.tgt, d.prob), devices={}).on(E.current_device())
    b = corpus.batch
    want = E.mine_host(dd, model, b, 2.0, 0.5, -1.0, 1.0, want_sim=True)
    f = {k: np.array(getattr(b, k), copy=True) for k in ("pair_src", "pair_tgt", "sent_len", "pair_sim_off")}
    k = 37  # a pair in the middle
    if fault == "src_past_end":
        f["pair_src"][k] = b.n_sentences - 1
    elif fault == "tgt_negative":
        f["pair_tgt"][k] = -5
    elif fault == "empty_sentence":
        f["sent_len"][int(b.pair_tgt[k]) + 1] = 0
    elif fault == "tokens_past_end":
        f["sent_len"][b.n_sentences - 1] += 1000  # the last sentence runs past the token array
    else:
        f["pair_sim_off"][k] = -1
    bad = dataclasses.replace(b, **f)
    with pytest.raises(BimineError):
        E.mine_host(dd, model, bad, 2.0, 0.5, -1.0, 1.0, want_sim=True)
    got = E.mine_host(dd, model, b, 2.0, 0.5, -1.0, 1.0, want_sim=True)
    assert np.array_equal(got[0], want[0])
    assert np.array_equal(got[1].view(np.uint8), want[1].view(np.uint8))
    assert bits_equal(got[2], want[2])


@pytest.mark.parametrize("pinned", [True, False])
def test_mine_host_narrow_wire_form(pinned):
    """bimine_mine_host with the compact wire form (24-bit token ids, uint16
    sentence arrays widened on the device) mines bit for bit what the int32
    form mines, from pinned and from pageable host arrays."""
    import torch

    from paper_1512_01641_b200.packing import PackedBatch

    corpus = synth.make_config(2, n_pairs=300)
    d = corpus.dictionary
    model = model_vector(H.synth_model())
    dd = E.LexiconContext(vocab=None, coo=(d.src, d.tgt, d.prob), devices={}).on(E.current_device())
    b = corpus.batch
    want = E.mine_host(dd, model, b, 2.0, 0.5, -1.0, 1.0, want_sim=True)
    wire = b.with_24bit_tokens().with_narrow_sentences()
    assert wire.sent_bytes == 2 and wire.token_bytes == 3
    if pinned:
        arrs = {f: torch.from_numpy(np.ascontiguousarray(getattr(wire, f))).pin_memory().numpy()
                for f in ("tokens", "sent_tok_off", "sent_len", "sent_uniq", "sent_chars", "pair_src", "pair_n",
                          "pair_tgt", "pair_m", "pair_sim_off")}
        wire = PackedBatch(**arrs, token_bytes=3, sent_bytes=2)
    got = E.mine_host(dd, model, wire, 2.0, 0.5, -1.0, 1.0, want_sim=True)
    assert np.array_equal(got[0], want[0])
    assert np.array_equal(got[1].view(np.uint8), want[1].view(np.uint8))
    assert bits_equal(got[2], want[2])


def test_mine_host_deterministic_across_calls():
    """Reruns are byte-identical (the reference's acceptance criterion 9,
    test_acceptance.py:279-326): 4,000 C2 pairs (~10M tokens, so the
    upload runs in several gated token pieces and the persistent score CTAs
    claim pairs in whatever order they land) mined eight times, alternating
    the int32 and the compact wire form."""
    corpus = synth.make_config(2, n_pairs=4_000)
    d = corpus.dictionary
    model = model_vector(H.synth_model())
    dd = E.LexiconContext(vocab=None, coo=(d.src, d.tgt, d.prob), devices={}).on(E.current_device())
    b = corpus.batch
    assert b.n_tokens > 8 << 20
    wire = b.with_24bit_tokens().with_narrow_sentences()
    first = E.mine_host(dd, model, b, 2.0, 0.5, -1.0, 1.0, want_sim=True)
    assert int(first[0].sum()) > 0
    for k in range(8):
        got = E.mine_host(dd, model, wire if k % 2 else b, 2.0, 0.5, -1.0, 1.0, want_sim=True)
        assert np.array_equal(got[0], first[0]), k
        assert np.array_equal(got[1].view(np.uint8), first[1].view(np.uint8)), k
        assert bits_equal(got[2], first[2]), k


def test_mine_host_concurrent_calls_one_device():
    """bimine_mine_host from several host threads on one device at once
    (pageable inputs: the staged upload path) gives every caller its own
    results -- calls on one device are serialised inside the library, so
    one call's waiting score CTAs never hold the SMs another call's upload
    pipeline needs."""
    from concurrent.futures import ThreadPoolExecutor

    d_list = []
    for seed in range(4):
        c = synth.make_config(2, seed_base=20261018 + 7 * seed, n_pairs=120 + 40 * seed)
        d_list.append(c)
    # one dictionary for all (the first corpus's), every batch mined with it
    d = d_list[0].dictionary
    model = model_vector(H.synth_model())
    dd = E.LexiconContext(vocab=None, coo=(d.src, d.tgt, d.prob), devices={}).on(E.current_device())
    batches = [c.batch if k % 2 else c.batch.with_24bit_tokens().with_narrow_sentences() for k, c in enumerate(d_list)]
    want = [E.mine_host(dd, model, b, 2.0, 0.5, -1.0, 1.0, want_sim=True) for b in batches]
    with ThreadPoolExecutor(4) as ex:
        got = list(ex.map(lambda b: E.mine_host(dd, model, b, 2.0, 0.5, -1.0, 1.0, want_sim=True), batches * 2))
    for k, g in enumerate(got):
        w = want[k % 4]
        assert np.array_equal(g[0], w[0])
        assert np.array_equal(g[1].view(np.uint8), w[1].view(np.uint8))
        assert bits_equal(g[2], w[2])


@pytest.mark.parametrize("chunks", ["3", "7"])
def test_mine_host_chunked_uploads(chunks):
    """bimine_mine_host with the batch uploaded in chunks (the score kernel
    waiting per chunk) gives the oracle's scores and matches, including a
    pair larger than one CTA (tiles) in the middle of the batch."""
    import subprocess, sys, os
    code = (
        "import sys; sys.path[:0]=['.','oracle','tests'];"
        "import numpy as np, helpers as H, oracle;"
        "from paper_1512_01641_b200 import synth, engine as E;"
        "from paper_1512_01641_b200.classifier import model_vector;"
        "from paper_1512_01641_b200.packing import BatchBuilder, Vocabulary;"
        "c=synth.make_config(2, n_pairs=40); d=c.dictionary; m=model_vector(H.synth_model());"
        "big=synth.make_config(1);"
        "ids=list(range(0,20))+[-1]+list(range(20,40));"
        "b=c.batch.select(list(range(40)));"
        "ctx=E.LexiconContext(vocab=None, coo=(d.src,d.tgt,d.prob), devices={});"
        "cnt,mt,sim=E.mine_host(ctx.on(0), m, b, 2.0, 0.5, -1.0, 1.0, want_sim=True);"
        "od=oracle.OracleDict(d.src,d.tgt,d.prob);"
        "ws=oracle.score_batch(od, m, b); wc,wr=oracle.mine_batch(od, m, b);"
        "assert np.array_equal(sim.view(np.uint64), ws.view(np.uint64));"
        "assert np.array_equal(cnt,wc); assert np.array_equal(mt.view(np.uint8), np.concatenate(wr).view(np.uint8));"
        "d1=big.dictionary; ctx1=E.LexiconContext(vocab=None, coo=(d1.src,d1.tgt,d1.prob), devices={});"
        "bb=big.batch; cnt1,mt1,sim1=E.mine_host(ctx1.on(0), m, bb, 2.0, 0.5, -1.0, 1.0, want_sim=True);"
        "od1=oracle.OracleDict(d1.src,d1.tgt,d1.prob); wc1,wr1=oracle.mine_batch(od1, m, bb);"
        "assert np.array_equal(cnt1,wc1); assert np.array_equal(mt1.view(np.uint8), np.concatenate(wr1).view(np.uint8));"
        "print('ok')"
    )
    env = dict(os.environ, BIMINE_E2E_CHUNKS=chunks, BIMINE_E2E_MIN_TOKENS="1")
    res = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600,
                         cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert res.returncode == 0 and "ok" in res.stdout, res.stderr[-3000:]


@pytest.mark.parametrize("shape", [(1500, 1700), (2100, 97), (96, 2100)])
def test_nw_large_problems_band_pipeline(shape):
    """Problems handled by the CTA-per-problem band pipeline (ring buffers
    between warps): steps, score and mined matches equal the oracle."""
    rng = np.random.default_rng(shape[0])
    sims = [rng.random(shape), (rng.random(shape) > 0.7).astype(np.float64)]
    out = E.nw_steps_host(sims, [1.3, 0.5], -1.0, 1.0)
    for sim, g, (codes, score) in zip(sims, [1.3, 0.5], out):
        want, _, _, want_score = oracle.nw_align(sim, -1.0, 1.0, g)
        assert np.array_equal(codes, want)
        assert bits_equal(score, want_score)
