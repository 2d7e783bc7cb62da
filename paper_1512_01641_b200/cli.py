"""``bimine mine`` / ``tune`` / ``dict`` on the GPU path.

Same positional arguments, options, defaults, outputs and exit codes as
the reference CLI for these two commands (cli.py:36-53, 157-230, 336-425):

    python -m paper_1512_01641_b200 mine CORPUS_DIR MODEL LEXICON OUT [--threshold ...]
    python -m paper_1512_01641_b200 tune CORPUS_DIR MODEL LEXICON REFERENCE [--budget ...]
    python -m paper_1512_01641_b200 dict PARALLEL OUT [--titles LINKS] [--iterations N]

``mine`` writes the bitext (``%.4f\\tsrc\\ttgt`` per mined pair, input
order) and ``OUT.manifest.json``, prints ``N sentence pairs mined from K
document pairs`` and reports failing pairs on stderr with exit status 1.
The scoring, DP, traceback and filtering run in libbimine_b200.so; the
engines ``nw`` and ``nw-wavefront`` are the same GPU path (their outputs
are identical by the reference's contract).  The A* engines are outside
this build's scope and are refused with a usage error.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

from . import __version__
from .align import MiningConfig, mine_corpus
from .classifier import load_model
from .corpus import load_corpus, read_links, read_parallel, write_bitext
from .lexicon import build_lexicon, merge_title_lexicon, read_lexicon, write_lexicon
from .manifest import RunManifest, file_digest, write_manifest

_ENGINES = {"nw": "nw", "nw-wavefront": "nw_wavefront"}
_OUT_OF_SCOPE = ("astar", "astar-unconstrained")


class UsageError(Exception):
    """Invalid command-line value: exit status 2 (argparse error)."""


def _engine_options(p: argparse.ArgumentParser) -> None:
    p.add_argument("--threshold", type=float, default=0.5)
    p.add_argument("--gap-penalty", type=float, default=2.0)
    p.add_argument("--match-bonus", type=float, default=1.0)
    p.add_argument("--mismatch-cost", type=float, default=-1.0)
    p.add_argument("--engine", choices=sorted(_ENGINES) + list(_OUT_OF_SCOPE), default="nw-wavefront")


def _manifest(args: argparse.Namespace, inputs: list[str], started: float) -> RunManifest:
    params = {k: v for k, v in sorted(vars(args).items()) if k not in ("func", "command") and not callable(v)}
    return RunManifest(command=args.command, parameters=params, inputs={p: file_digest(p) for p in inputs},
                       tool_version=__version__, wall_time_ms=int((time.perf_counter() - started) * 1000))


def _corpus_inputs(args) -> list[str]:
    return [os.path.join(args.corpus_dir, "pairs.tsv"), os.path.join(args.corpus_dir, "sentences.tsv"),
            args.model_file, args.lexicon_file]


def _check_engine(args) -> str:
    if args.engine in _OUT_OF_SCOPE:
        raise UsageError(f"engine {args.engine!r} is not part of the GPU path (A* search is out of scope)")
    return _ENGINES[args.engine]


def cmd_mine(args: argparse.Namespace) -> int:
    started = time.perf_counter()
    engine = _check_engine(args)
    pairs = load_corpus(args.corpus_dir)
    model = load_model(args.model_file)
    lexicon = read_lexicon(args.lexicon_file)
    config = MiningConfig(threshold=args.threshold, gap_penalty=args.gap_penalty, match_bonus=args.match_bonus,
                          mismatch_cost=args.mismatch_cost, workers=args.workers)
    outcome = mine_corpus(model, lexicon, pairs, config, engine=engine)
    write_bitext(args.out_file, outcome.rows)
    if args.verbose:
        hist: dict[str, int] = {}
        for score, _, _ in outcome.rows:
            key = f"{int(score * 10) / 10:.1f}"
            hist[key] = hist.get(key, 0) + 1
        for key in sorted(hist):
            print(f"score {key}x: {hist[key]} pairs")
    write_manifest(args.out_file + ".manifest.json", _manifest(args, _corpus_inputs(args), started))
    print(f"{len(outcome.rows)} sentence pairs mined from {len(pairs)} document pairs")
    if outcome.failures:
        for topic_id, error in outcome.failures:
            print(f"failed: {topic_id}: {error}", file=sys.stderr)
        print(f"{len(outcome.failures)} document pairs failed", file=sys.stderr)
        return 1
    return 0


def cmd_tune(args: argparse.Namespace) -> int:
    """cli.py:129-186: samples in corpus order with sorted reference indices,
    base config carrying --workers, seeded search, JSON report + manifest."""
    from .tuning import TuningSample, read_reference, tune

    started = time.perf_counter()
    engine = _check_engine(args)
    pairs = load_corpus(args.corpus_dir)
    model = load_model(args.model_file)
    lexicon = read_lexicon(args.lexicon_file)
    reference = read_reference(args.reference_file)
    topics = {p.topic_id for p in pairs}
    for topic_id in reference:
        if topic_id not in topics:
            raise ValueError(f"reference names unknown topic_id {topic_id!r}")
    samples = [TuningSample(pair=p, reference=tuple(sorted(reference[p.topic_id])))
               for p in pairs if p.topic_id in reference]
    result = tune(model, lexicon, samples, budget=args.budget, seed=args.seed, engine=engine,
                  base_config=MiningConfig(workers=args.workers))
    report = {
        "threshold": result.threshold, "gap_penalty": result.gap_penalty, "agreement": result.agreement,
        "trials": result.trials, "per_sample_agreement": list(result.per_sample),
        "default_agreement": result.default_agreement,
    }
    with open(args.out, "w", encoding="utf-8") as fh:
        json.dump(report, fh, indent=2, sort_keys=True)
        fh.write("\n")
    write_manifest(args.out + ".manifest.json",
                   _manifest(args, _corpus_inputs(args) + [args.reference_file], started))
    print(f"threshold={result.threshold:.4f} gap_penalty={result.gap_penalty:.4f} agreement={result.agreement:.2f}%")
    print(f"improvement over defaults: {result.agreement - result.default_agreement:.2f}%")
    return 0


def cmd_dict(args: argparse.Namespace) -> int:
    """cli.py:95-108: EM lexicon from sentence pairs (GPU rounds), optional
    title merge, sorted TSV + manifest."""
    started = time.perf_counter()
    lexicon = build_lexicon(read_parallel(args.parallel_file), args.iterations)
    inputs = [args.parallel_file]
    if args.titles:
        titles = read_links(args.titles)
        lexicon, skipped = merge_title_lexicon(lexicon, titles)
        inputs.append(args.titles)
        print(f"merged {len(titles) - skipped} title pairs, skipped {skipped}")
    write_lexicon(lexicon, args.out_file)
    write_manifest(args.out_file + ".manifest.json", _manifest(args, inputs, started))
    print(f"{len(lexicon)} lexicon entries written to {args.out_file}")
    return 0


def build_parser() -> argparse.ArgumentParser:
    common = argparse.ArgumentParser(add_help=False)
    common.add_argument("--seed", type=int, default=42)
    common.add_argument("--workers", type=int, default=1)
    common.add_argument("--verbose", action="store_true")
    parser = argparse.ArgumentParser(prog="bimine", description="Mine translation-equivalent sentence pairs (GPU path).")
    parser.add_argument("--version", action="version", version=f"%(prog)s {__version__}")
    sub = parser.add_subparsers(dest="command", required=True)
    p = sub.add_parser("dict", parents=[common], help="build the translation lexicon")
    p.add_argument("parallel_file")
    p.add_argument("out_file")
    p.add_argument("--titles")
    p.add_argument("--iterations", type=int, default=10)
    p.set_defaults(func=cmd_dict)
    p = sub.add_parser("mine", parents=[common], help="mine parallel sentences")
    for name in ("corpus_dir", "model_file", "lexicon_file", "out_file"):
        p.add_argument(name)
    _engine_options(p)
    p.set_defaults(func=cmd_mine)
    p = sub.add_parser("tune", parents=[common], help="tune threshold and gap penalty")
    for name in ("corpus_dir", "model_file", "lexicon_file", "reference_file"):
        p.add_argument(name)
    p.add_argument("--budget", type=int, default=100)
    p.add_argument("--engine", choices=sorted(_ENGINES) + ["astar"], default="nw-wavefront")
    p.add_argument("--out", default="tuning_report.json")
    p.set_defaults(func=cmd_tune)
    return parser


def main(argv: list[str] | None = None) -> int:
    parser = build_parser()
    args = parser.parse_args(argv)
    if args.command == "dict" and args.iterations < 1:
        parser.error("--iterations must be >= 1")
    if args.command == "tune" and args.budget < 1:
        parser.error("--budget must be >= 1")
    if args.workers < 1:
        parser.error("--workers must be >= 1")
    try:
        return args.func(args)
    except UsageError as exc:
        parser.error(str(exc))
        return 2
    except (ValueError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1
