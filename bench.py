"""Benchmark of the B200 sentence-alignment hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--pairs P]
    python bench.py --impl reference ...        # the CPU reference arm

A *step* is one mining pass over one batch of synthetic document pairs:
score kernel (build_score_matrix) -> NW wavefront fill + traceback +
threshold filter -> order-preserving compaction, with the packed batch
resident in HBM.  `value` is doc pairs/s over all ranks; NW GCUPS is
reported beside it.

Configs (BASELINE.json `configs`, index + 1):

* 2 (default) "C2": 10k pairs of ~50x50 sentences, 1M-entry dictionary,
  per rank -- weak scaling: each rank mines its own 10k pairs.
* 5 "C5": 1,000,000 pairs split over the N ranks by N*M cells -- strong
  scaling; the 1M pair descriptors are replicas of 10k generated pairs
  (sharing their sentences; generating 1M distinct pairs on the host would
  take ~20 min), each scored and aligned in full.
* 1, 3: the 200x220 pair and the 4096x4096 pair; 4: the tuning sweep.

`--gpus N` without torchrun re-launches this script under
`torch.distributed.run` with N ranks (one per GPU, NCCL only for the barrier
and the max-over-ranks timing); it exits non-zero if fewer than N GPUs are
visible.  The JSON line also carries `e2e` (the same metric through the C
ABI's host-buffer call bimine_mine_host: pinned H2D of the packed batch, all
kernels, D2H of counts + matches), `roofline` (score kernel vs measured HBM
peak and vs the issue-slot peak), `cpu_baseline` (N = 1, rank 0: the C port
of the reference path on a bounded sample, run in a subprocess; the
reference package's own `mine_corpus` and DP-only GCUPS beside it),
`per_rank` / `imbalance`, `clocks` and `gpu_launches`.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "doc pairs/s (score + NW + traceback/filter), NW GCUPS beside"
UNIT = "doc_pairs/s"
C5_TOTAL = 1_000_000
C5_BASE = 10_000


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4, 5],
                    help="BASELINE.json configs; 4 = the tuning sweep, 5 = 1M pairs strong scaling")
    ap.add_argument("--pairs", type=int, default=None,
                    help="pairs per rank (C1-C4) or in total (C5); default: the config's")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="target CPU-baseline sample duration")
    return ap.parse_args(argv)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def launch_ranks(args) -> int:
    """`--gpus N` outside torchrun: N ranks under torch.distributed.run."""
    import torch

    n = args.gpus
    visible = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if visible < n:
        print(json.dumps({"metric": METRIC, "error": f"--gpus {n}: only {visible} CUDA device(s) visible"}),
              flush=True)
        sys.stderr.write(f"bench.py: --gpus {n} needs {n} visible GPUs, found {visible}\n")
        return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__),
           *sys.argv[1:]]
    return subprocess.run(cmd).returncode


# ---------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------

def load_workload(config: int, pairs: int | None, rank: int):
    """(corpus, model vector) of a rank's C1-C4 batch (seeded per rank)."""
    from paper_1512_01641_b200 import synth
    from paper_1512_01641_b200.classifier import load_model, model_vector

    spec = synth.CONFIGS[config]
    n_pairs = pairs if pairs is not None else min(spec["n_pairs"], 10_000)
    rng_seed = 20261018
    dict_rng = np.random.default_rng(rng_seed + config)
    dictionary = synth.make_dictionary(dict_rng, spec["n_words"])
    corpus = synth.make_corpus(rng_seed + 1000 + config + 7919 * rank, n_pairs, spec["n_words"], spec["shape"],
                               dictionary=dictionary)
    model = model_vector(load_model(os.path.join(REPO, "tests", "golden", "synth_model.json")))
    return corpus, model


def c5_descriptors(base, total: int):
    """Pair shapes of C5's `total` descriptors: descriptor k is base pair k % B."""
    B = base.n_pairs
    idx = np.arange(total, dtype=np.int64) % B
    return idx, base.pair_n[idx].astype(np.int64) * base.pair_m[idx].astype(np.int64)


def c5_shard(base, total: int, rank: int, world: int):
    """Rank `rank`'s contiguous, cell-balanced share of C5's descriptors as a
    PackedBatch over the base batch's sentences; returns (batch, lo, hi)."""
    from paper_1512_01641_b200.distributed import shard_range
    from paper_1512_01641_b200.packing import PackedBatch

    idx, cells = c5_descriptors(base, total)
    lo, hi = shard_range(cells, rank, world)
    sel = idx[lo:hi]
    c = cells[lo:hi]
    sim_off = np.zeros(sel.shape[0], dtype=np.int64)
    if sel.shape[0] > 1:
        np.cumsum(c[:-1], out=sim_off[1:])
    batch = PackedBatch(tokens=base.tokens, sent_tok_off=base.sent_tok_off, sent_len=base.sent_len,
                        sent_uniq=base.sent_uniq, sent_chars=base.sent_chars, pair_src=base.pair_src[sel],
                        pair_n=base.pair_n[sel], pair_tgt=base.pair_tgt[sel], pair_m=base.pair_m[sel],
                        pair_sim_off=sim_off)
    return batch, lo, hi


def algorithmic_bytes(batch) -> int:
    """Score kernel's compulsory HBM traffic: the sim write,
    the token ids and the per-sentence / per-pair descriptors it reads.
    The dictionary (replicated, L2 resident) is excluded."""
    return int(8 * batch.n_cells + 4 * batch.n_tokens + 20 * batch.n_sentences + 48 * batch.n_pairs)


def _packed_offsets(batch) -> bool:
    """sent_tok_off == exclusive sum of sent_len (bimine_mine_host then skips its upload)."""
    want = np.zeros(batch.n_sentences, dtype=np.int64)
    np.cumsum(batch.sent_len[:-1], out=want[1:])
    return bool(np.array_equal(batch.sent_tok_off, want))


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        rows = []
        try:
            with open(self.path) as fh:
                for line in fh:
                    f = [x.strip() for x in line.split(",")]
                    if len(f) >= 9:
                        rows.append(f)
        finally:
            if self.path and os.path.exists(self.path):
                os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None

        sm = [num(r[1]) for r in rows if num(r[1]) is not None]
        smax = [num(r[2]) for r in rows if num(r[2]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k].lower() == "active"})
        return {
            "sm_mhz": statistics.median(sm) if sm else None,
            "sm_max_mhz": max(smax) if smax else None,
            "reasons": reasons,
            "samples": len(rows),
        }


def measured_peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        if d.get("hbm_gbs"):
            return float(d["hbm_gbs"]), float(d.get("sm_max_mhz") or 1965.0), "measured"
    except (OSError, ValueError):
        pass
    return 6650.0, 1965.0, "fallback"


def cpu_baselines(config: int, pairs: int | None, seconds: float, port_only: bool = False):
    """tools/ref_baseline.py in a subprocess: the C port (value) and, beside
    it, the reference package's own mine_corpus and DP GCUPS."""
    cmd = [sys.executable, os.path.join(REPO, "tools", "ref_baseline.py"), "--config", str(config),
           "--seconds", str(seconds)]
    if pairs is not None:
        cmd += ["--pairs", str(pairs)]
    if port_only:
        cmd.append("--port-only")
    try:
        res = subprocess.run(cmd, capture_output=True, text=True, timeout=max(300.0, 12 * seconds))
        line = [x for x in res.stdout.splitlines() if x.startswith("{")][-1]
        return json.loads(line)
    except (subprocess.SubprocessError, IndexError, ValueError) as exc:
        return {"error": f"ref_baseline failed: {exc}"}


def cpu_baseline_field(cb: dict):
    if "port" not in cb:
        return None
    out = dict(cb["port"])
    out["cpu_model"] = (cb.get("cpu") or {}).get("model")
    if "reference" in cb:
        out["reference_package"] = cb["reference"]
    return out


# ---------------------------------------------------------------------------
# the reference arm
# ---------------------------------------------------------------------------

def run_reference(args):
    """The reference path on the host cores (rank 0 only): the C port of the
    reference path (the line's value, conservative: faster than the
    reference's own Python path), with the reference package's own
    mine_corpus / DP GCUPS beside it."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    cfg = 2 if args.config == 5 else args.config
    per_step_s = 150.0 / (args.steps + args.warmup)
    cb = cpu_baselines(cfg, args.pairs, max(5.0, per_step_s))
    port = cb.get("port") or {}
    value = float(port.get("value", 0.0))
    batch_pairs = C5_TOTAL if args.config == 5 else (args.pairs or 10_000)
    dp = ((cb.get("reference") or {}).get("dp_gcups") or {})
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": args.gpus,  # the launch's N; the work runs on rank 0's host cores
        "steps": args.steps,
        "warmup": args.warmup,
        # a step = the config's batch (C2: 10k pairs) at the measured rate
        "ms_per_step": batch_pairs / value * 1e3 if value else None,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (SURVEY.md 8(d) generator, seeded)",
        "config": {"workload": f"C{args.config}" + (" (timed on C2 pairs: the same pair distribution)" if args.config == 5
                                                    else ""),
                   "devices": "host CPU only (rank 0)"},
        # DP-only GCUPS of the reference's compiled fill (kernels.fill_sequential,
        # its fastest backend here); the port's whole-pipeline cells/s beside it
        "nw_gcups": dp.get("fill_sequential"),
        "pipeline_gcups": (port.get("cells_per_s") or 0.0) / 1e9,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": port.get("cores"), "kind": "port",
                         "sample": port.get("sample"), "cpu_model": (cb.get("cpu") or {}).get("model"),
                         "reference_package": cb.get("reference")},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU arms
# ---------------------------------------------------------------------------

class Ranks:
    """Process group plumbing: barrier, max / all-gather of floats."""

    def __init__(self):
        import torch
        import torch.distributed as dist

        self.torch, self.dist = torch, dist
        self.rank, self.world, self.local = dist_env()
        if not torch.cuda.is_available() or torch.cuda.device_count() < 1:
            raise SystemExit("bench.py: no CUDA device visible")
        if self.world > 1:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{self.local}"))
        torch.cuda.set_device(self.local)
        self.dev = self.local

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def gather(self, values):
        t = self.torch.tensor(list(values), dtype=self.torch.float64, device=f"cuda:{self.dev}")
        if self.world == 1:
            return [t.tolist()]
        out = [self.torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t)
        return [o.tolist() for o in out]

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


def _roofline(alg_bytes, score_ms, instr_per_launch=None):
    hbm, sm_mhz, kind = measured_peaks()
    achieved = alg_bytes / (score_ms / 1e3) / 1e9
    out = {
        "kernel": "pair_kernel (score matrix), timed alone with CUDA events on the launching stream",
        "bound": "hbm",
        "achieved": achieved,
        "peak": hbm,
        "unit": "GB/s",
        "frac": achieved / hbm,
        "traffic": None,
        "peak_kind": f"{kind} (MEASURED_PEAKS.json hbm_gbs, burst copy)",
        "algorithmic_bytes_per_launch": alg_bytes,
        "launch_ms": score_ms,
    }
    return out


def _attach_traffic(roofline, workload_key):
    prof_traffic = os.path.join(REPO, "profiles", "score_kernel_traffic.json")
    if not os.path.exists(prof_traffic):
        return
    try:
        with open(prof_traffic) as fh:
            tr = json.load(fh)
        if tr.get("workload") == workload_key:
            roofline["traffic"] = tr.get("dram_bytes_per_launch")
            roofline["traffic_source"] = tr.get("source")
            if tr.get("warp_instructions_per_launch"):
                # issue-slot roofline beside the HBM one: the kernel is bound by
                # instruction issue (4 warp instructions / clock / SM peak)
                _, sm_mhz, _ = measured_peaks()
                peak = 148 * 4 * sm_mhz * 1e6
                ach = tr["warp_instructions_per_launch"] / (roofline["launch_ms"] / 1e3)
                roofline["issue"] = {"achieved_warp_instr_per_s": ach, "peak": peak, "frac": ach / peak,
                                     "warp_instructions_per_launch": tr["warp_instructions_per_launch"],
                                     "source": tr.get("source")}
    except (OSError, ValueError):
        pass


def time_mining(R, dd, model, batch, db, sim, steps, warmup, stream, gap, thr, mism, bonus):
    """K timed mining steps (L2 flushed between them): per-step ms of the
    mining launch and of the compaction, and the last output dict."""
    from paper_1512_01641_b200 import engine as E

    torch = R.torch
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{R.dev}")  # > 126 MB L2
    out = None

    def step(ev=None):
        nonlocal out
        out = E.mine_device(dd, model, db, sim, gap, thr, mism, bonus, out=out, stream=stream, events=ev)

    for _ in range(max(warmup, 3)):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    events = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
    R.barrier()
    torch.cuda.synchronize()
    with ClockSampler(R.dev) as clocks:
        for k in range(steps):
            flush.zero_()  # L2 flush between timed steps (outside the event window)
            step(events[k])
        torch.cuda.synchronize()
    R.barrier()
    mine_ms = sum(e[0].elapsed_time(e[1]) for e in events)
    compact_ms = sum(e[1].elapsed_time(e[2]) for e in events)
    return mine_ms, compact_ms, out, clocks.summary(), flush


def time_nw_and_score(R, dd, model, db, sim, out, steps, stream, flush, gap, thr, mism, bonus):
    from paper_1512_01641_b200 import engine as E

    torch = R.torch
    nw_out = dict(out)
    for _ in range(2):
        E.nw_device(db, sim, gap, thr, mism, bonus, nw_out, stream)
    nw_ms = 0.0
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for _ in range(steps):
        flush.zero_()
        ev[0].record(stream)
        E.nw_device(db, sim, gap, thr, mism, bonus, nw_out, stream)
        ev[1].record(stream)
        torch.cuda.synchronize()
        nw_ms += ev[0].elapsed_time(ev[1])
    for _ in range(2):
        E.score_device(dd, model, db, sim, stream)
    score_ms = 0.0
    for _ in range(steps):
        flush.zero_()
        ev[0].record(stream)
        E.score_device(dd, model, db, sim, stream)
        ev[1].record(stream)
        torch.cuda.synchronize()
        score_ms += ev[0].elapsed_time(ev[1])
    return nw_ms, score_ms


def pinned_batch(R, batch):
    """The batch's arrays copied into page-locked memory (a streaming
    caller's input buffers)."""
    from paper_1512_01641_b200.packing import PackedBatch

    pinned = {}
    for f in ("tokens", "sent_tok_off", "sent_len", "sent_uniq", "sent_chars", "pair_src", "pair_n",
              "pair_tgt", "pair_m", "pair_sim_off"):
        pinned[f] = R.torch.from_numpy(np.ascontiguousarray(getattr(batch, f))).pin_memory().numpy()
    return PackedBatch(**pinned, token_bytes=batch.token_bytes, sent_bytes=batch.sent_bytes)


def time_e2e(R, dd, model, batch, steps, warmup, stream, gap, thr, mism, bonus):
    """The same step end to end through bimine_mine_host: host batch in
    (pinned), counts + compacted matches out."""
    from paper_1512_01641_b200 import engine as E

    torch = R.torch
    pb = pinned_batch(R, batch)
    n_steps = max(20, steps) if batch.n_pairs <= 20_000 else max(3, steps)
    outbuf = {}  # a streaming caller's host output buffers, refilled every step
    for _ in range(max(3, warmup) if batch.n_pairs <= 20_000 else 1):
        E.mine_host(dd, model, pb, gap, thr, mism, bonus, stream=stream, out=outbuf)
    torch.cuda.synchronize()
    R.barrier()
    t0 = time.perf_counter()
    for _ in range(n_steps):
        counts, matches, _ = E.mine_host(dd, model, pb, gap, thr, mism, bonus, stream=stream, out=outbuf)
    e2e_s = time.perf_counter() - t0
    h2d = int(pb.nbytes()) - (8 * pb.n_sentences if _packed_offsets(pb) else 0)
    d2h = int(4 * batch.n_pairs + 8 + 16 * int(counts.sum()))
    return e2e_s, n_steps, h2d, d2h


def time_e2e_pageable(R, dd, model, batch, n_steps, stream, gap, thr, mism, bonus):
    """bimine_mine_host on the generator's own (pageable) numpy arrays: the
    library stages them through page-locked memory itself."""
    from paper_1512_01641_b200 import engine as E

    outbuf = {}
    E.mine_host(dd, model, batch, gap, thr, mism, bonus, stream=stream, out=outbuf)
    R.torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n_steps):
        E.mine_host(dd, model, batch, gap, thr, mism, bonus, stream=stream, out=outbuf)
    return time.perf_counter() - t0


def api_e2e(corpus, reps: int = 3):
    """The north-star interface end to end: align.mine_corpus from
    DocumentPairs (sentence text) to (score, src, tgt) rows, host
    tokenisation included, with a per-stage breakdown."""
    from paper_1512_01641_b200 import align as A
    from paper_1512_01641_b200.classifier import load_model
    from paper_1512_01641_b200.corpus import Document, DocumentPair
    from paper_1512_01641_b200.lexicon import Lexicon

    b = corpus.batch
    sents = corpus.all_sentences()
    pairs = []
    for p in range(b.n_pairs):
        s0, n, t0, m = int(b.pair_src[p]), int(b.pair_n[p]), int(b.pair_tgt[p]), int(b.pair_m[p])
        pairs.append(DocumentPair(f"t{p}", Document(f"s{p}", "pl", str(p), tuple(sents[s0:s0 + n])),
                                  Document(f"d{p}", "en", str(p), tuple(sents[t0:t0 + m]))))
    lex = Lexicon(corpus.dictionary.table())
    model = load_model(os.path.join(REPO, "tests", "golden", "synth_model.json"))
    cfg = A.MiningConfig()
    A.mine_corpus(model, lex, pairs[:64], cfg)  # lexicon upload, vocabulary, CUDA context: once per lexicon
    walls, stages = [], []
    for _ in range(reps):
        A.STAGE_TIMES = {}
        t0 = time.perf_counter()
        out = A.mine_corpus(model, lex, pairs, cfg)
        walls.append(time.perf_counter() - t0)
        stages.append(A.STAGE_TIMES)
    A.STAGE_TIMES = None
    k = int(np.argmin(walls))
    wall, st = walls[k], stages[k]
    return {
        "value": b.n_pairs / wall, "unit": UNIT, "pairs": b.n_pairs, "rows": len(out.rows),
        "path": "align.mine_corpus(model, lexicon, DocumentPairs, MiningConfig()) -> MiningOutcome rows "
                "(score, source sentence, target sentence)",
        "host_cores": os.cpu_count(), "chunk_pairs": A.CHUNK_PAIRS,
        "stages_s": {"tokenize_pack": st.get("pack", 0.0), "mine_host": st.get("mine", 0.0),
                     "rows": st.get("rows", 0.0),
                     "rest": max(0.0, wall - sum(st.values())), "total": wall},
    }


def run_gpu(args):
    """C1/C2/C3 (weak: every rank its own batch) and C5 (strong: 1M pairs
    split by N*M)."""
    from paper_1512_01641_b200 import engine as E

    R = Ranks()
    torch = R.torch
    strong = args.config == 5
    if strong:
        base, model = load_workload(5, C5_BASE, 0)
        total = args.pairs if args.pairs is not None else C5_TOTAL
        batch, lo, hi = c5_shard(base.batch, total, R.rank, R.world)
        d = base.dictionary
        workload = (f"C5: {total} doc pairs in total, split over {R.world} rank(s) by N*M cells "
                    f"(replicas of {C5_BASE} generated pairs sharing their sentences)")
    else:
        corpus, model = load_workload(args.config, args.pairs, R.rank)
        batch = corpus.batch
        d = corpus.dictionary
        total = batch.n_pairs * R.world
        lo, hi = 0, batch.n_pairs
        workload = (f"C{args.config}: {batch.n_pairs} doc pairs/rank, {batch.n_cells} cells, "
                    f"{batch.n_tokens} tokens, {len(d.src)}-entry dictionary")
    ctx = E.LexiconContext(vocab=None, coo=(d.src, d.tgt, d.prob), devices={})
    dd = ctx.on(R.dev)
    stream = torch.cuda.current_stream()
    db = E.DeviceBatch(batch, R.dev)
    sim = torch.empty(max(batch.n_cells, 1), dtype=torch.float64, device=f"cuda:{R.dev}")
    gap, thr, mism, bonus = 2.0, 0.5, -1.0, 1.0
    K = args.steps
    mine_ms, compact_ms, out, clocks, flush = time_mining(R, dd, model, batch, db, sim, K, args.warmup, stream,
                                                          gap, thr, mism, bonus)
    total_matches = int(out["total"].item())
    nw_ms, score_ms = time_nw_and_score(R, dd, model, db, sim, out, K, stream, flush, gap, thr, mism, bonus)
    del flush
    step_ms = mine_ms + compact_ms
    e2e = None
    e2e_pg = e2e_32 = 0.0
    h2d_32 = 0
    if not args.no_e2e:
        # the headline e2e uploads the compact wire form (24-bit ids, uint16
        # sentence arrays) when the values allow it; int32 arrays and
        # pageable inputs beside it
        wire = batch.with_24bit_tokens() if int(batch.tokens.max(initial=0)) < (1 << 24) else batch
        wire = wire.with_narrow_sentences()
        e2e_s, e2e_steps, h2d, d2h = time_e2e(R, dd, model, wire, K, args.warmup, stream, gap, thr, mism, bonus)
        if wire is not batch:
            e2e_32, _, h2d_32, _ = time_e2e(R, dd, model, batch, K, args.warmup, stream, gap, thr, mism, bonus)
        if not strong:
            e2e_pg = time_e2e_pageable(R, dd, model, batch, e2e_steps, stream, gap, thr, mism, bonus)
    else:
        e2e_s, e2e_steps, h2d, d2h = 0.0, 0, 0, 0
    per = R.gather([step_ms, mine_ms, nw_ms, score_ms, e2e_s, float(batch.n_pairs), float(batch.n_cells),
                    float(total_matches), e2e_pg, e2e_32])
    R.barrier()
    if R.rank != 0:
        R.close()
        return 0
    cols = list(zip(*per))
    step_max, mine_max, nw_max, score_max, e2e_max = (max(c) for c in cols[:5])
    pairs_all = sum(cols[5])
    cells_all = sum(cols[6])
    value = pairs_all * K / (step_max / 1e3)
    if not args.no_e2e:
        e2e = {
            "value": pairs_all * e2e_steps / e2e_max,
            "unit": UNIT,
            "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h,
            "steps": e2e_steps,
            "path": "bimine_mine_host (C ABI): pinned host inputs in the compact wire form (24-bit token ids, "
                    "bimine_batch.token_bytes = 3; uint16 sentence lengths / distinct counts / characters, "
                    "sent_bytes = 2), results copied into reused page-locked host output buffers"
                    + ("; per rank: the shared base sentences + its pair descriptors" if strong else ""),
        }
        if e2e_32:
            e2e["int32_tokens"] = {"value": pairs_all * e2e_steps / max(cols[9]), "h2d_bytes_per_step": h2d_32,
                                   "path": "the same call with int32 token ids and int32 sentence arrays"}
        if e2e_pg:
            e2e["pageable_inputs"] = {"value": pairs_all * e2e_steps / max(cols[8]),
                                      "path": "bimine_mine_host on the generator's pageable numpy arrays (staged "
                                              "through page-locked memory inside the library)"}
    plan = db.plan
    nw_launches = (1 if plan.n_large < batch.n_pairs else 0) + (3 if plan.n_large else 0)
    launches_per_step = 1 + (plan.n_long > 0) + nw_launches + 2
    roofline = None
    if R.world == 1 and not strong:
        roofline = _roofline(algorithmic_bytes(batch), score_max / K)
        _attach_traffic(roofline, f"C{args.config}:{batch.n_pairs}")
    api = None
    if R.world == 1 and not strong and args.config == 2 and not args.no_e2e:
        api = api_e2e(corpus)
    cpu = None
    if R.world == 1 and not args.no_cpu:
        # C3 (one 4096x4096 pair): the C port alone (~1 min on 16 threads);
        # the reference package's Python mine_corpus would take hours
        cpu = cpu_baseline_field(cpu_baselines(2 if strong else args.config, None if strong else args.pairs,
                                               args.cpu_seconds, port_only=args.config == 3))
    line = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": R.world,
        "steps": K,
        "warmup": max(args.warmup, 3),
        "ms_per_step": step_max / K,
        "higher_is_better": True,
        "scaling": "strong" if strong else "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (SURVEY.md 8(d) generator, seeded; model trained by the reference's train_classifier)",
        "config": {
            "workload": workload,
            "pairs_total": int(pairs_all),
            "cells_total": int(cells_all),
            "mining": {"threshold": thr, "gap_penalty": gap, "match_bonus": bonus, "mismatch_cost": mism},
            "l2": "flushed (512 MB write) between timed steps",
            "parallelism": f"pair shards x{R.world}, no collective on the data path",
        },
        "nw_gcups": cells_all * K / (nw_max / 1e3) / 1e9,
        "pipeline_gcups": cells_all * K / (step_max / 1e3) / 1e9,
        "mine_ms_per_step": mine_max / K,
        "nw_only_ms": nw_max / K,
        "score_only_ms": score_max / K,
        "matches_per_step": int(sum(cols[7])),
        "per_rank": {"step_ms": [c[0] / K for c in per], "pairs": [int(c[5]) for c in per],
                     "cells": [int(c[6]) for c in per]},
        "imbalance": (max(cols[0]) / (sum(cols[0]) / len(cols[0]))) if cols[0] else None,
        "e2e": e2e,
        "api_e2e": api,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "clocks": clocks,
        "gpu_launches": launches_per_step * K,
    }
    print(json.dumps(line), flush=True)
    R.close()
    return 0


TUNE_SETTINGS = 64


def _tuning_inputs(corpus):
    from paper_1512_01641_b200.align import MiningConfig
    from paper_1512_01641_b200.tuning import draw_trials

    thresholds, gaps = draw_trials(MiningConfig(), TUNE_SETTINGS, seed=7)
    refs = [[tuple(map(int, x)) for x in r] for r in corpus.reference]
    return thresholds, gaps, refs


def _cpu_tuning(corpus, model, thresholds, gaps, refs, n_pairs, threads):
    """The reference's tune() per sample (tuning.py:92-153) restated on the
    C oracle: score once, then per setting NW + traceback + filter and the
    agreement NW (0/1 equality matrix, gap 1, bonus 1, mismatch -1)."""
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import oracle

    oracle.build()
    d = corpus.dictionary
    od = oracle.OracleDict(d.src, d.tgt, d.prob)
    sample = corpus.batch.select(range(n_pairs))
    t0 = time.perf_counter()
    sims = oracle.score_batch(od, model, sample, threads)
    for p in range(n_pairs):
        n, m = int(sample.pair_n[p]), int(sample.pair_m[p])
        sim = sims[sample.pair_sim_off[p]: sample.pair_sim_off[p] + n * m].reshape(n, m)
        ref = refs[p]
        for thr, gap in zip(thresholds, gaps):
            codes, _, _, _ = oracle.nw_align(sim, -1.0, 1.0, gap)
            i = j = 0
            cand = []
            for c in codes:
                if c == 0:
                    if sim[i, j] >= thr:
                        cand.append((i, j))
                    i += 1
                    j += 1
                elif c == 1:
                    i += 1
                else:
                    j += 1
            if ref and cand:
                eq = np.array([[1.0 if a == b else 0.0 for b in ref] for a in cand])
                oracle.nw_align(eq, -1.0, 1.0, 1.0)
    return n_pairs / (time.perf_counter() - t0), sample.n_cells


def run_tuning(args):
    """C4: one step = the tuning sweep over the batch -- score every pair
    once, align it under all 64 (threshold, gap) settings in one batched NW
    launch (problem = pair x setting), agreement NW of every candidate list
    against the reference on device.  value = doc pairs tuned per second."""
    from paper_1512_01641_b200 import engine as E

    rank, world, _ = dist_env()
    if args.impl == "reference":
        if rank != 0:
            return 0
        corpus, model = load_workload(4, args.pairs, 0)
        thresholds, gaps, refs = _tuning_inputs(corpus)
        sys.path.insert(0, os.path.join(REPO, "oracle"))
        import oracle

        threads = oracle.max_threads()
        probe_rate, _ = _cpu_tuning(corpus, model, thresholds, gaps, refs, 2, threads)
        n = max(1, min(corpus.batch.n_pairs, int(probe_rate * 150.0 / (args.steps + args.warmup))))
        rates = [_cpu_tuning(corpus, model, thresholds, gaps, refs, n, threads)[0] for _ in range(args.steps)]
        value = float(np.mean(rates))
        print(json.dumps({
            "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": n / value * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (SURVEY.md 8(d) generator, seeded)",
            "config": {"workload": f"C4: tuning sweep, {TUNE_SETTINGS} settings", "sample_pairs_per_step": n},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": f"{n} pairs x {TUNE_SETTINGS} settings per step: oracle score (OpenMP) + "
                                       "per-setting NW/filter/agreement (1 thread)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }), flush=True)
        return 0
    R = Ranks()
    torch = R.torch
    corpus, model = load_workload(4, args.pairs, R.rank)
    batch = corpus.batch
    thresholds, gaps, refs = _tuning_inputs(corpus)
    d = corpus.dictionary
    dd = E.LexiconContext(vocab=None, coo=(d.src, d.tgt, d.prob), devices={}).on(R.dev)
    stream = torch.cuda.current_stream()
    P, S = batch.n_pairs, TUNE_SETTINGS
    tuner = E.DeviceTuner(dd, model, batch, thresholds, gaps, -1.0, 1.0, refs, stream=stream)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{R.dev}")
    for _ in range(max(args.warmup, 3)):
        flush.zero_()
        tuner.run_device()
    torch.cuda.synchronize()
    events = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    R.barrier()
    torch.cuda.synchronize()
    with ClockSampler(R.dev) as clocks:
        for k in range(args.steps):
            flush.zero_()
            tuner.run_device(events=events[k])
        torch.cuda.synchronize()
    R.barrier()
    parts = [sum(e[i].elapsed_time(e[i + 1]) for e in events) for i in range(3)]
    K = args.steps
    e2e_s, e2e_steps = 0.0, 0
    if not args.no_e2e:
        for _ in range(max(3, args.warmup)):  # warm (allocator growth, first touches)
            E.tune_device(dd, model, batch, thresholds, gaps, -1.0, 1.0, refs, tuner=tuner)
        torch.cuda.synchronize()
        R.barrier()
        e2e_steps = max(20, K)
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            E.tune_device(dd, model, batch, thresholds, gaps, -1.0, 1.0, refs, tuner=tuner)
        e2e_s = time.perf_counter() - t0
    per = R.gather([sum(parts)] + parts + [e2e_s])
    if R.rank != 0:
        R.close()
        return 0
    cols = list(zip(*per))
    step_ms, score_ms, nw_ms, agree_ms, e2e_max = (max(c) for c in cols)
    value = P * R.world * K / (step_ms / 1e3)
    e2e = None
    if not args.no_e2e:
        e2e = {"value": P * R.world * e2e_steps / e2e_max, "unit": UNIT, "h2d_bytes_per_step": int(batch.nbytes()),
               "d2h_bytes_per_step": 8 * P * S, "steps": e2e_steps,
               "path": "engine.tune_device: host batch in (pinned upload into the tuner's persistent device "
                       "batch), per-(pair, setting) counts + agreements out"}
    cpu = None
    if R.world == 1 and not args.no_cpu:
        sys.path.insert(0, os.path.join(REPO, "oracle"))
        import oracle

        threads = oracle.max_threads()
        rate, cells = _cpu_tuning(corpus, model, thresholds, gaps, refs, min(P, 40), threads)
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"first {min(P, 40)} pairs x {S} settings: oracle score ({threads} OpenMP threads) + "
                         "per-setting NW/filter/agreement (1 thread)"}
    nw_alg = 8.25 * batch.n_cells * S  # sim read + 2-bit directions per cell and setting
    peak, _, peak_kind = measured_peaks()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": R.world, "steps": K, "warmup": args.warmup,
        "ms_per_step": step_ms / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (SURVEY.md 8(d) generator, seeded; model trained by the reference's "
                                "train_classifier; settings drawn as tune() draws them, seed 7)",
        "config": {"workload": f"C4: tuning sweep, {P} doc pairs/rank x {S} (threshold, gap) settings",
                   "pairs_per_rank": P, "settings": S, "cells_per_rank": int(batch.n_cells),
                   "l2": "flushed (512 MB write) between timed steps",
                   "parallelism": f"pair shards x{R.world}, no collective on the data path"},
        "score_ms_per_step": score_ms / K, "nw_ms_per_step": nw_ms / K, "agreement_ms_per_step": agree_ms / K,
        "nw_gcups": batch.n_cells * S * K / (nw_ms / 1e3) / 1e9,
        "e2e": e2e,
        "roofline": {"kernel": "nw_kernel (64 settings x 1k pairs, one warp per problem)", "bound": "hbm",
                     "achieved": nw_alg / (nw_ms / K / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                     "frac": nw_alg / (nw_ms / K / 1e3) / 1e9 / peak, "traffic": None,
                     "peak_kind": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)",
                     "algorithmic_bytes_per_launch": nw_alg,
                     "note": "sim (20 MB) is re-read 64x from L2, so the DP is latency/issue bound"},
        "cpu_baseline": cpu, "clocks": clocks.summary(), "gpu_launches": 3 * K,
    }
    print(json.dumps(line), flush=True)
    R.close()
    return 0


def main(argv=None):
    args = parse(argv)
    rank, world, _ = dist_env()
    if world > 1 and args.gpus != world and args.impl == "b200":
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}\n")
        return 2
    if world == 1 and args.gpus > 1 and args.impl == "b200":
        return launch_ranks(args)
    if args.config == 4:
        return run_tuning(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
