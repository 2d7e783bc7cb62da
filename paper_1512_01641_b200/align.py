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

``mine_corpus`` tokenises and packs the pairs in chunks (pairs whose
sentences do not tokenise, or that a device limit rejects, are reported as
failures with the reference's message and skipped, align.py:396-399/441-447),
mines chunk k on GPU k mod min(config.workers, visible GPUs) while the next
chunk is packed; output order is input order for every worker count.  The A* engines (align.py:203-320) are not
part of the GPU path: requesting them raises ``NotImplementedError``.
"""

from __future__ import annotations

import contextlib
import gc
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import engine as _engine
from .classifier import model_vector
from .packing import BatchBuilder, PackedBatch, pack_documents

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


CHUNK_PAIRS = 5_000  # pairs tokenised / mined per chunk of mine_corpus (the next chunk packs while one mines)
# stage timer of mine_corpus (bench.py's api_e2e): None, or a dict that
# accumulates seconds per stage -- "pack" (tokenise + pack), "mine"
# (bimine_mine_host), "rows" (result tuples)
STAGE_TIMES: dict | None = None


def _stage(name: str, t0: float) -> None:
    if STAGE_TIMES is not None:
        STAGE_TIMES[name] = STAGE_TIMES.get(name, 0.0) + time.perf_counter() - t0


def _chunk_bounds(n: int, min_chunks: int) -> list[tuple[int, int]]:
    k = max(min_chunks, -(-n // CHUNK_PAIRS), 1)
    k = min(k, max(n, 1))
    cuts = [n * c // k for c in range(k + 1)]
    return [(a, b) for a, b in zip(cuts[:-1], cuts[1:]) if b > a]


def _mine_chunk(model, lexicon, pd, config: MiningConfig, device: int, topic_ids, lo: int):
    """Mine one packed chunk on `device`; returns (rows, failures) of the
    chunk, rows in input order.  A device-side limit (BimineError) must not
    abort the corpus: the chunk is then mined pair by pair and the pairs
    that still fail are reported (align.py:396-399, 441-447)."""
    import torch

    from ._native import BimineError

    keep = np.flatnonzero(pd.ok)
    failed: dict[int, str] = {}
    t0 = time.perf_counter()
    with torch.cuda.device(device):
        try:
            counts, matches = _mine_packed(model, lexicon, pd.batch, config, device=device)
            counts = counts.astype(np.int64)
        except BimineError:
            counts, parts = np.zeros(keep.size, dtype=np.int64), []
            for b in range(keep.size):
                try:
                    c, m = _mine_packed(model, lexicon, pd.batch.select([b]), config, device=device)
                    counts[b] = int(c[0])
                    parts.append(m.copy())
                except BimineError as exc:
                    failed[lo + int(keep[b])] = f"pair {topic_ids[lo + int(keep[b])]}: {exc}"
            matches = np.concatenate(parts) if parts else np.zeros(0, dtype=_native_match_dtype())
    _stage("mine", t0)
    # rows: every match's sentences by index into the chunk's sentence list
    # (built natively, csrc/pyhost.c: ~10^5 - 10^7 tuples)
    if matches.shape[0] == 0:
        return [], failed
    t0 = time.perf_counter()
    from .packing import _pyhost

    rows = _pyhost().build_rows(np.ascontiguousarray(matches), np.ascontiguousarray(counts, dtype=np.int64),
                                keep.astype(np.int64), pd.docs)
    _stage("rows", t0)
    return rows, failed


def _native_match_dtype():
    from . import _native as N

    return N.MATCH_DTYPE


def mine_corpus(model, lexicon, pairs: Sequence, config: MiningConfig, engine: str = "nw_wavefront") -> MiningOutcome:
    """Mine document pairs; output follows input order for any ``workers``.

    The pairs are tokenised and packed in chunks (the next chunk is packed on
    the host while the previous ones mine on the GPUs); ``config.workers``
    sets the minimum number of chunks ("shards"), which go round-robin to
    the visible GPUs, one host thread per device.  Results are assembled in
    input order.  Failing pairs -- untokenisable sentences, or a document a
    device limit rejects -- are reported and skipped, never raised.
    """
    _check_engine(engine)
    with _no_gc():  # the rows are ~10^5 - 10^7 fresh tuples: no collector passes while they are built
        return _mine_corpus(model, lexicon, pairs, config)


@contextlib.contextmanager
def _no_gc():
    was = gc.isenabled()
    gc.disable()
    try:
        yield
    finally:
        if was:
            gc.enable()


def _mine_corpus(model, lexicon, pairs: Sequence, config: MiningConfig) -> MiningOutcome:
    ctx = _engine.lexicon_context(lexicon)
    n = len(pairs)
    import torch

    _engine.current_device()  # loud: no library or no GPU
    n_dev = max(1, min(config.workers, torch.cuda.device_count()))
    chunks = _chunk_bounds(n, config.workers)
    topic_ids = [p.topic_id for p in pairs]
    errors: dict[int, str] = {}
    pools = [ThreadPoolExecutor(max_workers=1) for _ in range(n_dev)]  # a device's chunks in order
    futures = []
    try:
        for c, (lo, hi) in enumerate(chunks):
            t0 = time.perf_counter()
            pd = pack_documents(ctx.vocab, [(p.source.sentences, p.target.sentences) for p in pairs[lo:hi]])
            _stage("pack", t0)
            for k, msg in pd.errors.items():
                errors[lo + k] = f"pair {topic_ids[lo + k]}: {msg}"
            if pd.batch is None:
                continue
            futures.append(pools[c % n_dev].submit(_mine_chunk, model, lexicon, pd, config, c % n_dev, topic_ids,
                                                   lo))
        rows: list[tuple[float, str, str]] = []
        for fut in futures:
            chunk_rows, failed = fut.result()
            rows.extend(chunk_rows)
            errors.update(failed)
    finally:
        for pool in pools:
            pool.shutdown(wait=True)
    failures = tuple((topic_ids[k], errors[k]) for k in sorted(errors))
    return MiningOutcome(rows=tuple(rows), failures=failures)
