"""File-level drop-in for `bimine mine` / `bimine tune`.

CPU: the corpus directory, bitext and field escaping against the files the
reference wrote (tests/golden/cli, made by tests/golden/make_golden.py).
GPU: the CLI itself against the reference CLI's bitext bytes, printed
lines, exit codes and tuning report.
"""

import contextlib
import io
import json
import os
import shutil

import pytest

from paper_1512_01641_b200 import cli
from paper_1512_01641_b200 import corpus as C

HERE = os.path.dirname(os.path.abspath(__file__))
G = os.path.join(HERE, "golden", "cli")
MODEL = os.path.join(HERE, "golden", "synth_model.json")


def _expect():
    with open(os.path.join(G, "expect.json")) as fh:
        return json.load(fh)


def test_escape_round_trip_kats():
    for raw, esc in [("a\tb", "a\\tb"), ("x\\y", "x\\\\y"), ("l\nm", "l\\nm"), ("\\t", "\\\\t"), ("plain", "plain")]:
        assert C.escape_field(raw) == esc
        assert C.unescape_field(esc) == raw


def test_load_corpus_reads_reference_files(tmp_path):
    pairs = C.load_corpus(os.path.join(G, "corpus"))
    assert len(pairs) == 10
    assert pairs[3].topic_id == "cli\\3"  # escaped backslash
    assert pairs[5].source.title == "tab\there"  # escaped tab
    assert "..." in pairs[7].target.sentences
    assert all(p.source.lang == "pl" and p.target.lang == "en" for p in pairs)
    C.save_corpus(pairs, tmp_path / "again")
    for name in ("pairs.tsv", "sentences.tsv"):
        assert (tmp_path / "again" / name).read_bytes() == open(os.path.join(G, "corpus", name), "rb").read()


def test_bitext_round_trip(tmp_path):
    src = os.path.join(G, "mined_default.tsv")
    rows = C.read_bitext(src)
    assert rows and all(0.0 <= s <= 1.0 for s, _, _ in rows)
    C.write_bitext(tmp_path / "b.tsv", rows)
    assert (tmp_path / "b.tsv").read_bytes() == open(src, "rb").read()
    (tmp_path / "bad.tsv").write_text("0.5\tonly two\n")
    with pytest.raises(ValueError, match="line 1: expected 3 tab-separated fields, got 2"):
        C.read_bitext(tmp_path / "bad.tsv")


def test_cli_usage_errors(tmp_path, capsys):
    with pytest.raises(SystemExit) as ex:
        cli.main(["mine", G, MODEL, "lex", str(tmp_path / "o"), "--workers", "0"])
    assert ex.value.code == 2
    with pytest.raises(SystemExit) as ex:  # A* search is outside the GPU path
        cli.main(["mine", os.path.join(G, "corpus"), MODEL, os.path.join(G, "lexicon.tsv"), str(tmp_path / "o"),
                  "--engine", "astar"])
    assert ex.value.code == 2
    assert cli.main(["mine", str(tmp_path / "missing"), MODEL, "lex", str(tmp_path / "o")]) == 1
    assert "error:" in capsys.readouterr().err


def _run(argv):
    so, se = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(so), contextlib.redirect_stderr(se):
        rc = cli.main(argv)
    return rc, so.getvalue(), se.getvalue()


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["default", "strict"])
def test_cli_mine_matches_reference_bytes(tmp_path, name):
    want = _expect()[f"mine_{name}"]
    out = tmp_path / "mined.tsv"
    rc, so, se = _run(["mine", os.path.join(G, "corpus"), MODEL, os.path.join(G, "lexicon.tsv"), str(out),
                       *want["argv"]])
    assert (rc, so, se) == (want["rc"], want["stdout"], want["stderr"])
    assert out.read_bytes() == open(os.path.join(G, f"mined_{name}.tsv"), "rb").read()
    man = json.load(open(str(out) + ".manifest.json"))
    assert man["command"] == "mine" and len(man["inputs"]) == 4


@pytest.mark.gpu
def test_cli_tune_matches_reference(tmp_path):
    want = _expect()["tune"]
    good = tmp_path / "good"
    pairs = [p for k, p in enumerate(C.load_corpus(os.path.join(G, "corpus"))) if k != 7]
    C.save_corpus(pairs, good)
    rep = tmp_path / "report.json"
    rc, so, se = _run(["tune", str(good), MODEL, os.path.join(G, "lexicon.tsv"), os.path.join(G, "reference.tsv"),
                       "--budget", "8", "--seed", "3", "--out", str(rep)])
    assert (rc, so) == (want["rc"], want["stdout"])
    assert json.load(open(rep)) == want["report"]


@pytest.mark.gpu
def test_cli_dict_matches_reference_bytes(tmp_path):
    """`dict`: EM rounds on the GPU + title merge + sorted TSV, byte-identical
    to the reference CLI's lexicon file and printed lines."""
    want = _expect()["dict"]
    out = tmp_path / "lex.tsv"
    rc, so, se = _run(["dict", os.path.join(G, "parallel.tsv"), str(out), "--titles", os.path.join(G, "titles.tsv")])
    assert (rc, so.replace(str(out), "<OUT>"), se) == (want["rc"], want["stdout"], want["stderr"])
    assert out.read_bytes() == open(os.path.join(G, "dict_lexicon.tsv"), "rb").read()


def test_read_parallel_errors(tmp_path):
    (tmp_path / "p.tsv").write_text("a\tb\n\nc\td\te\n")
    with pytest.raises(ValueError, match="line 3: expected 2 tab-separated fields, got 3"):
        C.read_parallel(tmp_path / "p.tsv")
    assert C.read_links(os.path.join(G, "titles.tsv"))[0][0] == "s0"
