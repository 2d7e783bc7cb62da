"""CPU-only checks of the host side: tokenizer, packing, the exp
restatement, the C ABI surface, configuration and sharding logic."""

import ctypes
import dataclasses
import os
import re
import subprocess
import sys

import numpy as np
import pytest

import helpers as H
from paper_1512_01641_b200 import align as A
from paper_1512_01641_b200 import synth
from paper_1512_01641_b200.packing import BatchBuilder, PackedBatch, Vocabulary, unique_counts
from paper_1512_01641_b200.text import tokenize

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(REPO, "paper_1512_01641_b200", "csrc")
HEADER = os.path.join(REPO, "include", "bimine_b200.h")


def test_tokenize_matches_reference_rules():
    # text.py:97-104: lower, split on whitespace, strip ASCII punctuation
    assert tokenize("Domo, kato!") == ["domo", "kato"]
    assert tokenize("...") == []
    assert tokenize("  A\tb\nC  ") == ["a", "b", "c"]
    assert tokenize("(dog) -- x.y 'z'") == ["dog", "x.y", "z"]
    assert tokenize("Żółw «ok»") == ["żółw", "«ok»"]  # non-ASCII punctuation is kept
    assert tokenize("ǅ") == ["ǆ"]


def test_batch_builder_profiles_and_errors():
    vocab = Vocabulary()
    b = BatchBuilder(vocab)
    b.add_pair(["a b a.", "Żółw!"], ["b c", "a"])
    with pytest.raises(ValueError, match="target sentence 1: untokenizable sentence: '...'"):
        b.add_pair(["a"], ["b", "..."])
    with pytest.raises(ValueError, match="both sentence sequences must be non-empty"):
        b.add_pair([], ["b"])
    pb = b.build()
    assert pb.n_pairs == 1 and pb.n_sentences == 4
    assert pb.sent_len.tolist() == [3, 1, 2, 1]
    assert pb.sent_uniq.tolist() == [2, 1, 2, 1]
    assert pb.sent_chars.tolist() == [len("a b a."), len("Żółw!"), 3, 1]
    assert pb.pair_src.tolist() == [0] and pb.pair_tgt.tolist() == [2]
    assert pb.pair_sim_off.tolist() == [0] and pb.n_cells == 4
    assert [vocab.words[t] for t in pb.tokens.tolist()] == ["a", "b", "a", "żółw", "b", "c", "a"]


def test_unique_counts_and_select():
    corpus = synth.make_config(2, n_pairs=5)
    b = corpus.batch
    want = [len(set(b.tokens[o : o + l].tolist())) for o, l in zip(b.sent_tok_off, b.sent_len)]
    assert unique_counts(b.tokens, b.sent_len).tolist() == want
    sub = b.select([3, 1])
    assert sub.n_pairs == 2
    assert sub.pair_n.tolist() == [b.pair_n[3], b.pair_n[1]]
    s3 = b.tokens[b.sent_tok_off[b.pair_src[3]] : b.sent_tok_off[b.pair_src[3]] + b.sent_len[b.pair_src[3]]]
    assert np.array_equal(sub.tokens[: len(s3)], s3)


def test_synthetic_generator_is_deterministic_and_shaped():
    a = synth.make_config(2, n_pairs=20)
    b = synth.make_config(2, n_pairs=20)
    assert np.array_equal(a.batch.tokens, b.batch.tokens)
    assert a.batch.pair_n.min() >= 40 and a.batch.pair_n.max() <= 60
    assert np.all(np.abs(a.batch.pair_m - a.batch.pair_n) <= 5)
    assert a.batch.sent_len.min() >= 1
    assert 3 <= np.median(a.batch.sent_len) <= 40
    assert len(a.dictionary.src) > 900_000  # ~1M-entry dictionary
    for p, ref in enumerate(a.reference):
        assert all(i2 > i1 and j2 > j1 for (i1, j1), (i2, j2) in zip(ref, ref[1:]))
    src, tgt = a.pair_sentences(0)
    assert len(src) == a.batch.pair_n[0] and all(s.endswith(".") for s in src)


def test_exp_table_matches_definition():
    sys.path.insert(0, CSRC)
    import gen_exp_table

    with open(os.path.join(CSRC, "exp_table.inc")) as fh:
        assert fh.read() == gen_exp_table.render()


def test_host_compiled_exp_matches_libm(tmp_path):
    """glibc_exp.cuh compiled for the host equals libm exp (math.exp)."""
    src = tmp_path / "t.cpp"
    src.write_text(
        '#include "%s/glibc_exp.cuh"\n#include <cstdio>\n#include <random>\n#include <cmath>\n'
        "int main(){std::mt19937_64 g(3);long bad=0;std::uniform_real_distribution<double> u(-750,720);\n"
        "for(long i=0;i<3000000;++i){double x=i%%3?u(g):bimine::u2d(g());double a=bimine::glibc_exp(x,bimine::kExpTable),b=exp(x);\n"
        "if(bimine::d2u(a)!=bimine::d2u(b)&&!(std::isnan(a)&&std::isnan(b)))++bad;}printf(\"%%ld\\n\",bad);return bad!=0;}\n" % CSRC
    )
    exe = tmp_path / "t"
    subprocess.run(["g++", "-O2", "-ffp-contract=off", "-std=c++17", str(src), "-o", str(exe), "-lm"], check=True)
    res = subprocess.run([str(exe)], capture_output=True, text=True)
    assert res.returncode == 0, res.stdout


def _declared_symbols():
    with open(HEADER) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\**\s*(bimine_[a-z_0-9]+)\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    from paper_1512_01641_b200 import _native, build

    build.build()
    L = _native.load(require_gpu=False)
    declared = _declared_symbols()
    assert len(declared) >= 14
    for name in declared:
        assert hasattr(L, name), name
        assert name in _native.SIGNATURES, name
    assert L.bimine_version().startswith(b"bimine_b200")
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True, text=True).stdout
    for name in declared:
        assert re.search(rf"\bT {name}$", out, re.M), name


def test_library_is_sm100a():
    from paper_1512_01641_b200 import _native

    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_product_path_fails_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1512_01641_b200 import _native

    with pytest.raises(_native.NativeUnavailable):
        A.build_score_matrix(H.toy_model(), H.toy_lexicon(), ["domo"], ["house"])
    with pytest.raises(_native.NativeUnavailable):
        A.nw_align(np.eye(3), A.MiningConfig())


def test_config_and_engine_validation():
    with pytest.raises(ValueError):
        A.MiningConfig(threshold=1.5)
    with pytest.raises(ValueError):
        A.MiningConfig(gap_penalty=-0.1)
    with pytest.raises(ValueError):
        A.MiningConfig(workers=0)
    with pytest.raises(ValueError, match="unknown engine"):
        A.mine_corpus(None, None, [], A.MiningConfig(), engine="bogus")
    with pytest.raises(NotImplementedError):
        A.mine_corpus(None, None, [], A.MiningConfig(), engine="astar_constrained")
    with pytest.raises(ValueError):
        A.nw_align(np.zeros((0, 3)), A.MiningConfig())
    with pytest.raises(ValueError):
        A.nw_align(np.array([[np.nan]]), A.MiningConfig())


def test_filter_by_threshold_kat():
    sim = np.array([[0.9, 0.0, 0.0], [0.0, 0.4, 0.0], [0.0, 0.0, 0.7]])
    al = A.Alignment(steps=(A.Match(0, 0), A.Match(1, 1), A.Match(2, 2)), score=0.0)
    assert A.filter_by_threshold(sim, al, 0.5) == [(0.9, 0, 0), (0.7, 2, 2)]


def test_steps_from_codes():
    steps = A._steps_from_codes(np.array([0, 1, 2, 0, 2], dtype=np.uint8))
    assert steps == (A.Match(0, 0), A.GapSource(1), A.GapTarget(1), A.Match(2, 2), A.GapTarget(3))


def test_shard_bounds_cover_in_order():
    w = np.array([5, 1, 1, 8, 2, 2, 2, 9, 1], dtype=np.int64)
    for parts in (1, 2, 3, 4, 8, 20):
        b = A._shard_bounds(w, parts)
        assert b[0][0] == 0 and b[-1][1] == len(w)
        assert all(x[1] == y[0] for x, y in zip(b, b[1:]))
        assert len(b) <= parts


def _native_vocab():
    from paper_1512_01641_b200 import build
    from paper_1512_01641_b200.packing import NativeVocabulary

    build.build()
    return NativeVocabulary()


def test_native_tokenizer_matches_python_rules():
    """bimine_tokenize_batch == text.tokenize (text.py:97-104) on ASCII and,
    through the Python path, on non-ASCII sentences; same vocabulary ids."""
    import random

    v = _native_vocab()
    rng = random.Random(5)
    alphabet = "abcXYZ019 .,;:!?'\"()[]-_\t\n\x0b\x0c\r\x1c\x1d\x1e\x1f\x00~`@#$%^&*+=<>/\\|{}"
    sents = ["".join(rng.choice(alphabet) for _ in range(rng.randint(0, 40))) for _ in range(3000)]
    sents += ["Żółw «ok» x", "ǅ ab", "naïve café.", " a　b\x85c", "İstanbul"]
    tokens, lens, uniq, chars = v.tokenize(sents)
    pos = 0
    for s, L, U, C in zip(sents, lens.tolist(), uniq.tolist(), chars.tolist()):
        want = tokenize(s)
        got = tokens[pos : pos + L].tolist()
        pos += L
        assert [v.get(w) for w in want] == got, s
        assert U == len(set(want)) and C == len(s)
    assert pos == tokens.shape[0]


def test_native_tokenizer_in_place_list():
    """bimine_tokenize_ptrs over the sentences' own str storage (_pyhost.str_view)
    == text.tokenize, on a list large enough to be
    split over threads, with words of 1-40 bytes (the 8/16-byte key
    boundaries and the long-word path) and words ending at the last byte;
    a list holding a non-ASCII str or a str subclass takes the UTF-8 path
    with the same ids."""
    import random

    from paper_1512_01641_b200.packing import _pyhost

    v = _native_vocab()
    rng = random.Random(11)
    letters = "abcdefghijklmnopqrstuvwxyzABCDEFGHIJKLMNOPQRSTUVWXYZ0123456789"
    punct = ".,;:!?'\"()[]-_"
    space = " \t\n\x0b\x0c\r\x1c\x1d\x1e\x1f"

    def sentence():
        parts = []
        for _ in range(rng.randint(0, 30)):
            w = "".join(rng.choice(letters) for _ in range(rng.choice([1, 2, 7, 8, 9, 15, 16, 17, 24, 40])))
            if rng.random() < 0.2:
                w = rng.choice(punct) + w + rng.choice(punct) * rng.randint(1, 3)
            parts.append(w + "".join(rng.choice(space) for _ in range(rng.randint(1, 2))))
        s = "".join(parts)
        return s if rng.random() < 0.5 else s.rstrip()

    sents = [sentence() for _ in range(20000)]
    assert sum(map(len, sents)) > 2 << 20  # several thread ranges
    n = len(sents)
    ptrs, lens, prefix = np.empty(n, np.int64), np.empty(n, np.int64), np.empty(n + 1, np.int64)
    assert _pyhost().str_view(sents, ptrs, lens, prefix)
    assert prefix[n] == sum(map(len, sents)) and lens.tolist() == list(map(len, sents))

    class S(str):
        pass

    def check(batch):
        tokens, lens, uniq, chars = v.tokenize(batch)
        pos = 0
        for s, L, U, C in zip(batch, lens.tolist(), uniq.tolist(), chars.tolist()):
            want = tokenize(s)
            got = tokens[pos : pos + L].tolist()
            pos += L
            assert [v.get(w) for w in want] == got, repr(s)
            assert U == len(set(want)) and C == len(s)
        assert pos == tokens.shape[0]

    check(sents)
    check(["a b c d e f g"] * 3000 + ["x"])  # denser than one token per 5 characters: the retry
    for odd in ("na\u00efve x", S("subclass str")):
        batch = sents[:3000] + [odd] + sents[3000:6000]
        m = len(batch)
        assert not _pyhost().str_view(batch, np.empty(m, np.int64), np.empty(m, np.int64), np.empty(m + 1, np.int64))
        check(batch)


def test_build_rows_matches_python():
    """_pyhost.build_rows (csrc/pyhost.c) == the rows built in Python
    (align.py:441-447: (score, source sentence, target sentence) per match,
    pair by pair), the same str objects; bad inputs raise."""
    from paper_1512_01641_b200 import _native as N
    from paper_1512_01641_b200.packing import _pyhost

    _native_vocab()  # builds _pyhost too
    rng = np.random.default_rng(3)
    K = 40
    docs = [(tuple(f"s{k}.{i}" for i in range(rng.integers(1, 6))), [f"t{k}.{j}" for j in range(rng.integers(1, 6))])
            for k in range(K)]
    pair = np.sort(rng.choice(K, 30, replace=False)).astype(np.int64)
    counts = np.array([rng.integers(0, min(len(docs[k][0]), len(docs[k][1])) + 1) for k in pair], np.int64)
    m = np.empty(int(counts.sum()), dtype=N.MATCH_DTYPE)
    want, r = [], 0
    for k, c in zip(pair.tolist(), counts.tolist()):
        for _ in range(c):
            i, j = rng.integers(0, len(docs[k][0])), rng.integers(0, len(docs[k][1]))
            m[r] = (rng.random(), i, j)
            want.append((float(m[r]["score"]), docs[k][0][i], docs[k][1][j]))
            r += 1
    got = _pyhost().build_rows(m, counts, pair, docs)
    assert got == want and all(g[1] is w[1] and g[2] is w[2] for g, w in zip(got, want))
    assert _pyhost().build_rows(m[:0], np.zeros(30, np.int64), pair, docs) == []
    with pytest.raises(ValueError):  # counts do not cover the matches
        _pyhost().build_rows(m, counts + 1, pair, docs)
    bad = m.copy()
    bad["i"] += 10
    with pytest.raises(IndexError):  # a sentence index past the pair
        _pyhost().build_rows(bad, counts, pair, docs)
    with pytest.raises(TypeError):  # a pair index past the list
        _pyhost().build_rows(m, counts, pair + K, docs)


def test_docs_view_matches_flat_view():
    """_pyhost.docs_view over (source, target) pairs == str_view over the
    flattened sentences; any other shape or a non-ASCII str -> False."""
    from paper_1512_01641_b200.packing import _pyhost

    _native_vocab()
    docs = [(("a b", "c"), ["dd", "e f g"]), (["h"], ("i", "j", "k"))]
    flat = [s for d in docs for side in d for s in side]
    n = len(flat)
    out = [np.empty(n, np.int64), np.empty(n, np.int64), np.empty(n + 1, np.int64)]
    ref = [np.empty(n, np.int64), np.empty(n, np.int64), np.empty(n + 1, np.int64)]
    start = np.array([0, 4, 8], np.int64)
    assert _pyhost().docs_view(docs, *out, start) and _pyhost().str_view(flat, *ref)
    assert all((a == b).all() for a, b in zip(out, ref))
    many = docs * 3000  # several thread ranges
    fm = [s for d in many for side in d for s in side]
    st = np.arange(0, 4 * len(many) + 1, 4, dtype=np.int64)
    o2 = [np.empty(len(fm), np.int64), np.empty(len(fm), np.int64), np.empty(len(fm) + 1, np.int64)]
    r2 = [np.empty(len(fm), np.int64), np.empty(len(fm), np.int64), np.empty(len(fm) + 1, np.int64)]
    assert _pyhost().docs_view(many, *o2, st) and _pyhost().str_view(fm, *r2)
    assert all((a == b).all() for a, b in zip(o2, r2))
    bad_counts = st.copy()
    bad_counts[5] += 1
    assert not _pyhost().docs_view(many, *o2, bad_counts)
    for odd in ([(("a",), ("\u00e9",))], [(("a",),)], [("a", "b")], [(("a",), ("b",), ("c",))]):
        assert not _pyhost().docs_view(odd, np.empty(4, np.int64), np.empty(4, np.int64), np.empty(5, np.int64),
                                       np.array([0, 2], np.int64))


def test_narrow_sentence_form():
    """PackedBatch.with_narrow_sentences: uint16 copies of the three sentence
    arrays with bimine_batch.sent_bytes = 2 (values unchanged); a batch with
    a value of 2^16 or more stays int32; the entry points other than
    bimine_mine_host refuse the narrow form (bimine_plan_batch here)."""
    from paper_1512_01641_b200 import _native as N
    from paper_1512_01641_b200 import engine as E

    _native_vocab()
    b = synth.make_config(2, n_pairs=30).batch
    nb = b.with_narrow_sentences()
    assert nb.sent_bytes == 2 and nb.with_narrow_sentences() is nb
    for f in ("sent_len", "sent_uniq", "sent_chars"):
        assert getattr(nb, f).dtype == np.uint16
        assert np.array_equal(getattr(nb, f).astype(np.int64), getattr(b, f).astype(np.int64))
    assert N.batch_struct_host(nb).sent_bytes == 2 and N.batch_struct_host(b).sent_bytes == 4
    wide = dataclasses.replace(b, sent_chars=b.sent_chars.copy())
    wide.sent_chars[3] = 70000
    assert wide.with_narrow_sentences() is wide
    with pytest.raises(N.BimineError, match="sent_bytes = 2"):
        E.plan_batch(nb)


def test_utf8_offsets_edge_cases():
    """The UTF-8 packing behind bimine_tokenize_batch: bytes back to back and
    byte offsets, for ASCII, non-ASCII, empty strings, NULs and lone
    surrogates (surrogatepass, as NativeVocabulary.add_many encodes)."""
    from paper_1512_01641_b200.packing import _utf8_offsets

    cases = [[], [""], ["", ""], ["abc", "", "d"], ["żółw", "", "x\x00y", "ó"], ["\udc80", "a\ud800b"],
             ["ascii"] * 3 + ["ĄĘ"], [chr(c) for c in range(1, 0x800, 7)]]
    for strs in cases:
        data, off = _utf8_offsets(strs)
        enc = [x.encode("utf-8", "surrogatepass") for x in strs]
        assert data == b"".join(enc), strs
        assert off.tolist() == [0] + np.cumsum([len(e) for e in enc]).tolist(), strs


def test_native_tokenizer_latin_range_exhaustive(monkeypatch):
    """Every code point below U+0180, inside words, alone and at token
    edges: the native Latin path equals CPython's lower()/split()/strip()
    (text.py:97-104) and len(text); only U+0130 (lowers to two code points)
    is left to the Python rules."""
    from paper_1512_01641_b200 import packing

    v = _native_vocab()
    sents = [f"A{chr(c)}b {chr(c)} .{chr(c)}, Ż{chr(c)}Ó" for c in range(1, 0x180)]
    fallback = []
    real = packing.tokenize

    def spy(s):
        fallback.append(s)
        return real(s)

    monkeypatch.setattr(packing, "tokenize", spy)
    tokens, lens, uniq, chars = v.tokenize(sents)
    pos = 0
    for s, L, U, C in zip(sents, lens.tolist(), uniq.tolist(), chars.tolist()):
        want = tokenize(s)
        assert [v.get(w) for w in want] == tokens[pos: pos + L].tolist(), repr(s)
        assert U == len(set(want)) and C == len(s), repr(s)
        pos += L
    assert fallback == [f"A{chr(0x130)}b {chr(0x130)} .{chr(0x130)}, Ż{chr(0x130)}Ó"]


def test_native_tokenizer_polish_text_stays_native(monkeypatch):
    import random

    from paper_1512_01641_b200 import packing

    v = _native_vocab()
    rng = random.Random(7)
    words = ["Zażółć", "gęślą", "jaźń", "ŁÓDŹ", "świeże", "Kraków", "ĄĘ", "über", "Straße", "Ÿ", "naïve", "x"]
    sents = [" ".join(rng.choice(words) + rng.choice(["", ",", ".", "!"]) for _ in range(rng.randint(1, 12)))
             + rng.choice(["", "\xa0", "\x85 tail"]) for _ in range(500)]
    seen = []
    monkeypatch.setattr(packing, "tokenize", lambda s: seen.append(s) or tokenize(s))
    tokens, lens, uniq, chars = v.tokenize(sents)
    assert seen == []
    pos = 0
    for s, L, C in zip(sents, lens.tolist(), chars.tolist()):
        assert [v.get(w) for w in tokenize(s)] == tokens[pos: pos + L].tolist(), repr(s)
        assert C == len(s)
        pos += L


def test_native_tokenizer_threaded_batch():
    """A batch past the multi-thread split (>= 512 KB): same tokens as the
    Python rules, long words sharing their first 16 bytes kept apart, and
    ids assigned in first-occurrence order as by one serial pass."""
    import random

    from paper_1512_01641_b200.packing import NativeVocabulary

    _native_vocab()
    rng = random.Random(11)
    words = [f"w{k}" for k in range(5000)] + [f"internationalisation{k}x" for k in range(300)]
    words += ["".join(rng.choice("abcdefghijklmnopqrstuvwxyz") for _ in range(rng.randint(1, 30))) for _ in range(3000)]

    def sentence():
        out = []
        for _ in range(rng.randint(1, 30)):
            w = rng.choice(words)
            w = w.upper() if rng.random() < 0.1 else w
            out.append(rng.choice(["", "(", '"']) + w + rng.choice(["", ",", ".", "!?"]))
        return rng.choice([" ", "  ", "\t"]).join(out)

    sents = [sentence() for _ in range(9000)]
    assert sum(map(len, sents)) > 1 << 20
    v = NativeVocabulary()
    tokens, lens, uniq, chars = v.tokenize(sents)
    first = list(dict.fromkeys(tokens.tolist()))
    assert first == list(range(len(first))) == list(range(len(v)))
    sents[100:100] = ["Żółw INTERNATIONALISATION7X w1", "ǅ w2."]  # Python-rule sentences in the same batch
    tokens, lens, uniq, chars = v.tokenize(sents)
    pos = 0
    for s, L, U, C in zip(sents, lens.tolist(), uniq.tolist(), chars.tolist()):
        want = tokenize(s)
        assert [v.get(w) for w in want] == tokens[pos : pos + L].tolist(), s
        assert U == len(set(want)) and C == len(s)
        pos += L
    assert pos == tokens.shape[0]


def test_native_and_python_builders_agree():
    from paper_1512_01641_b200.packing import BatchBuilder, Vocabulary

    corpus = synth.make_config(2, n_pairs=4)
    pairs = [corpus.pair_sentences(p) for p in range(4)]
    pairs.insert(2, (["ok s1."], ["...", "t2"]))  # untokenizable target sentence
    pairs.insert(3, ([], ["t2"]))
    nb = BatchBuilder(_native_vocab())
    pb = BatchBuilder(Vocabulary())
    rn = nb.add_pairs(pairs)
    rp = pb.add_pairs(pairs)
    assert rn == rp
    assert rn[2] == "target sentence 0: untokenizable sentence: '...'"
    assert rn[3] == "both sentence sequences must be non-empty"
    a, b = nb.build(), pb.build()
    for f in ("sent_len", "sent_uniq", "sent_chars", "pair_src", "pair_n", "pair_tgt", "pair_m", "pair_sim_off"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    # ids differ between vocabularies only by renaming: compare token strings
    pv = pb.vocab.words
    inv = {}
    for w in set(pv):
        inv[nb.vocab.get(w)] = w
    assert [inv[t] for t in a.tokens.tolist()] == [pv[t] for t in b.tokens.tolist()]


def test_24bit_token_form_round_trip():
    from paper_1512_01641_b200 import synth

    b = synth.make_config(2, n_pairs=20).batch
    p = b.with_24bit_tokens()
    assert p.token_bytes == 3 and p.tokens.dtype == np.uint8 and p.tokens.size == 3 * b.n_tokens
    assert p.n_tokens == b.n_tokens and p.nbytes() == b.nbytes() - b.n_tokens
    assert np.array_equal(p.int32_tokens(), b.tokens)
    edge = dataclasses.replace(b, tokens=np.array([0, 1, (1 << 24) - 1, 1 << 23, 255, 256] +
                                                  [7] * (b.n_tokens - 6), dtype=np.int32))
    assert np.array_equal(edge.with_24bit_tokens().int32_tokens(), edge.tokens)
    for bad in (-1, 1 << 24):
        with pytest.raises(ValueError):
            dataclasses.replace(b, tokens=np.full(b.n_tokens, bad, dtype=np.int32)).with_24bit_tokens()
