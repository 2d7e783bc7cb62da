"""Public alignment / mining API -- drop-in for ``bimine.align``.

Same names, signatures, defaults, error messages and ordering contracts
as the reference (pkg/src/bimine/align.py:45-448); the work runs on the
GPU through libbimine_b200.so:

* ``build_score_matrix``  (align.py:102-129)  -> score kernel
* ``nw_align`` / ``nw_align_wavefront`` (align.py:170-200) -> NW wavefront
  kernel in step mode (both engines are the same GPU wavefront; the
  reference guarantees their outputs are identical, align.py:184-187)
* ``align_pair_indices`` / ``mine_document_pair`` / ``mine_corpus``
  (align.py:347-448) -> one ``bimine_mine_host`` call per batch: score
  kernel, NW + traceback + threshold filter, compaction in input order
  (uploads overlapped with the scoring).

``mine_corpus`` packs all pairs into one batch (pairs whose sentences do
not tokenise are reported as failures with the reference's message and
skipped, align.py:396-399/441-447) and shards pairs over
``min(config.workers, visible GPUs)`` devices; output order is input
order for every worker count.  The A* engines (align.py:203-320) are not
part of the GPU path: requesting them raises ``NotImplementedError``.
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import engine as _engine
from .classifier import model_vector
from .packing import BatchBuilder, PackedBatch

ENGINES = ("nw", "nw_wavefront", "astar_constrained")
GPU_ENGINES = ("nw", "nw_wavefront")


@dataclass(frozen=True)
class Match:
    i: int
    j: int


@dataclass(frozen=True)
class GapSource:
    i: int


@dataclass(frozen=True)
class GapTarget:
    j: int


Step = Match | GapSource | GapTarget


@dataclass(frozen=True)
class Alignment:
    steps: tuple[Step, ...]
    score: float


@dataclass(frozen=True)
class MiningConfig:
    """Threshold, gap penalty and the affine map of scores (align.py:73-90)."""

    threshold: float = 0.5
    gap_penalty: float = 2.0
    match_bonus: float = 1.0
    mismatch_cost: float = -1.0
    workers: int = 1

    def __post_init__(self) -> None:
        if not 0.0 <= self.threshold <= 1.0:
            raise ValueError("threshold must lie in [0, 1]")
        if self.gap_penalty < 0.0:
            raise ValueError("gap penalty must be >= 0")
        if self.workers < 1:
            raise ValueError("workers must be >= 1")


@dataclass(frozen=True)
class MiningOutcome:
    rows: tuple[tuple[float, str, str], ...]
    failures: tuple[tuple[str, str], ...]  # (topic_id, error message)


def _validate_scores(scores) -> np.ndarray:
    sim = np.asarray(scores, dtype=np.float64)
    if sim.ndim != 2 or sim.shape[0] == 0 or sim.shape[1] == 0:
        raise ValueError("score matrix must be a non-empty 2-D array")
    if not np.all(np.isfinite(sim)) or sim.min() < 0.0 or sim.max() > 1.0:
        raise ValueError("score matrix values must be finite and lie in [0, 1]")
    return sim


def _check_engine(engine_name: str) -> None:
    if engine_name not in ENGINES:
        raise ValueError(f"unknown engine {engine_name!r}; expected one of {ENGINES}")
    if engine_name not in GPU_ENGINES:
        raise NotImplementedError(
            f"engine {engine_name!r} (best-first search) is not part of the B200 path; use 'nw' or 'nw_wavefront'"
        )


def build_score_matrix(model, lexicon, source_sentences: Sequence[str], target_sentences: Sequence[str]) -> np.ndarray:
    """Similarity of every source sentence against every target sentence."""
    if not source_sentences or not target_sentences:
        raise ValueError("both sentence sequences must be non-empty")
    ctx = _engine.lexicon_context(lexicon)
    batch = _pack_one(ctx.vocab, source_sentences, target_sentences)
    dd = ctx.on(_engine.current_device())
    flat = _engine.score_host(dd, model_vector(model), batch)
    return flat.reshape(len(source_sentences), len(target_sentences))


def _pack_one(vocab, source, target) -> PackedBatch:
    """One pair through the (native) tokenizer; the reference's ValueError
    messages (align.py:109-119) for empty or untokenizable input."""
    builder = BatchBuilder(vocab)
    [res] = builder.add_pairs([(source, target)])
    if isinstance(res, str):
        raise ValueError(res)
    return builder.build()


def _steps_from_codes(codes: np.ndarray) -> tuple[Step, ...]:
    steps: list[Step] = []
    i = j = 0
    for c in codes.tolist():
        if c == 0:
            steps.append(Match(i, j))
            i += 1
            j += 1
        elif c == 1:
            steps.append(GapSource(i))
            i += 1
        else:
            steps.append(GapTarget(j))
            j += 1
    return tuple(steps)


def _nw(scores, config: MiningConfig) -> Alignment:
    sim = _validate_scores(scores)
    [(codes, score)] = _engine.nw_steps_host([sim], [config.gap_penalty], config.mismatch_cost, config.match_bonus)
    return Alignment(steps=_steps_from_codes(codes), score=score)


def nw_align(scores, config: MiningConfig, backend: str | None = None) -> Alignment:
    """Optimal monotone alignment by dynamic programming (GPU wavefront)."""
    return _nw(scores, config)


def nw_align_wavefront(scores, config: MiningConfig, workers: int, backend: str | None = None) -> Alignment:
    """Anti-diagonal fill of the same table; identical output to ``nw_align``."""
    if workers < 1:
        raise ValueError("workers must be >= 1")
    return _nw(scores, config)


def nw_align_batch(matrices: Sequence[np.ndarray], config: MiningConfig) -> list[Alignment]:
    """nw_align over many matrices in one GPU launch."""
    sims = [_validate_scores(s) for s in matrices]
    if not sims:
        return []
    out = _engine.nw_steps_host(sims, [config.gap_penalty] * len(sims), config.mismatch_cost, config.match_bonus)
    return [Alignment(steps=_steps_from_codes(c), score=s) for c, s in out]


def astar_align(scores, config: MiningConfig, constrained: bool = True) -> Alignment:
    raise NotImplementedError("best-first (A*) alignment is not part of the B200 path; use nw_align")


def filter_by_threshold(scores, alignment: Alignment, threshold: float) -> list[tuple[float, int, int]]:
    """Match steps whose similarity reaches the threshold, in step order."""
    sim = np.asarray(scores)
    return [
        (float(sim[s.i, s.j]), s.i, s.j)
        for s in alignment.steps
        if isinstance(s, Match) and sim[s.i, s.j] >= threshold
    ]


def run_engine(scores, config: MiningConfig, engine: str, wavefront_workers: int = 1) -> Alignment:
    if engine == "nw":
        return nw_align(scores, config)
    if engine == "nw_wavefront":
        return nw_align_wavefront(scores, config, wavefront_workers)
    if engine == "astar_constrained":
        return astar_align(scores, config, constrained=True)
    raise ValueError(f"unknown engine {engine!r}; expected one of {ENGINES}")


def _mine_packed(model, lexicon, batch: PackedBatch, config: MiningConfig, device: int | None = None):
    """(counts, matches) of a packed batch on one device."""
    ctx = _engine.lexicon_context(lexicon)
    dd = ctx.on(_engine.current_device() if device is None else device)
    counts, matches, _ = _engine.mine_host(
        dd, model_vector(model), batch, config.gap_penalty, config.threshold, config.mismatch_cost, config.match_bonus
    )
    return counts, matches


def align_pair_indices(model, lexicon, pair, config: MiningConfig, engine: str = "nw_wavefront",
                       wavefront_workers: int = 1) -> list[tuple[float, int, int]]:
    """Mine one document pair down to (score, i, j) index triples."""
    _check_engine(engine)
    if wavefront_workers < 1:
        raise ValueError("workers must be >= 1")
    src, tgt = pair.source.sentences, pair.target.sentences
    if not src or not tgt:
        raise ValueError("both sentence sequences must be non-empty")
    batch = _pack_one(_engine.lexicon_context(lexicon).vocab, src, tgt)
    counts, matches = _mine_packed(model, lexicon, batch, config)
    return [(float(r["score"]), int(r["i"]), int(r["j"])) for r in matches]


def mine_document_pair(model, lexicon, pair, config: MiningConfig, engine: str = "nw_wavefront",
                       wavefront_workers: int = 1) -> list[tuple[float, str, str]]:
    """Mined sentence pairs of one document pair, with similarity scores."""
    try:
        matches = align_pair_indices(model, lexicon, pair, config, engine, wavefront_workers)
    except ValueError as exc:
        raise ValueError(f"pair {pair.topic_id}: {exc}") from None
    return [(score, pair.source.sentences[i], pair.target.sentences[j]) for score, i, j in matches]


def _shard_bounds(weights: np.ndarray, parts: int) -> list[tuple[int, int]]:
    """Contiguous ranges of near-equal total weight (N*M cells per pair)."""
    n = weights.shape[0]
    if parts <= 1 or n == 0:
        return [(0, n)]
    c = np.cumsum(weights, dtype=np.float64)
    cuts = [0]
    for k in range(1, parts):
        cuts.append(int(np.searchsorted(c, c[-1] * k / parts, side="left")))
    cuts.append(n)
    cuts = sorted(set(max(0, min(n, x)) for x in cuts))
    return [(a, b) for a, b in zip(cuts[:-1], cuts[1:]) if b > a]


def mine_corpus(model, lexicon, pairs: Sequence, config: MiningConfig, engine: str = "nw_wavefront") -> MiningOutcome:
    """Mine document pairs; output follows input order for any ``workers``.

    ``config.workers`` > 1 shards the pairs over that many visible GPUs
    (contiguous ranges balanced by cell count, one host thread per
    device); results are concatenated in shard order, which is input
    order.  Failing pairs are reported and skipped.
    """
    _check_engine(engine)
    ctx = _engine.lexicon_context(lexicon)
    builder = BatchBuilder(ctx.vocab)
    index_of: list[int] = []  # batch pair -> input pair
    errors: dict[int, str] = {}
    results = builder.add_pairs([(p.source.sentences, p.target.sentences) for p in pairs])
    for k, (pair, res) in enumerate(zip(pairs, results)):
        if isinstance(res, str):
            errors[k] = f"pair {pair.topic_id}: {res}"
        else:
            index_of.append(k)
    batch = builder.build()
    per_pair: list = [None] * len(pairs)
    if batch.n_pairs:
        import torch

        n_dev = max(1, min(config.workers, torch.cuda.device_count()))
        weights = batch.pair_n.astype(np.int64) * batch.pair_m.astype(np.int64)
        shards = _shard_bounds(weights, n_dev)

        def run(shard_dev):
            (lo, hi), dev = shard_dev
            sub = batch if (lo, hi) == (0, batch.n_pairs) else batch.select(range(lo, hi))
            with torch.cuda.device(dev):
                counts, matches = _mine_packed(model, lexicon, sub, config, device=dev)
            return lo, counts, matches

        jobs = [(s, d) for d, s in enumerate(shards)]
        if len(jobs) == 1:
            results = [run(jobs[0])]
        else:
            with ThreadPoolExecutor(max_workers=len(jobs)) as ex:
                results = list(ex.map(run, jobs))
        for lo, counts, matches in results:
            score, ii, jj = matches["score"].tolist(), matches["i"].tolist(), matches["j"].tolist()
            pos = 0
            for b, c in enumerate(counts.tolist()):
                per_pair[index_of[lo + b]] = (score[pos : pos + c], ii[pos : pos + c], jj[pos : pos + c])
                pos += c
    rows: list[tuple[float, str, str]] = []
    failures: list[tuple[str, str]] = []
    for k, pair in enumerate(pairs):
        if k in errors:
            failures.append((pair.topic_id, errors[k]))
            continue
        src, tgt = pair.source.sentences, pair.target.sentences
        score, ii, jj = per_pair[k]
        rows.extend(zip(score, [src[i] for i in ii], [tgt[j] for j in jj]))
    return MiningOutcome(rows=tuple(rows), failures=tuple(failures))
