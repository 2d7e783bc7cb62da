"""CPU baselines for bench.py, run in a SUBPROCESS so the GPU arm's process
never loads a checker or the reference (its native_so list stays the
product's own library).

    python tools/ref_baseline.py --config 2 [--seconds 15] [--port-only]

Prints one JSON object:

* ``port``: the C oracle (oracle/bimine_oracle.c, our plain-C restatement of
  the reference path) mining a bounded prefix of the workload on all host
  threads -- doc pairs/s;
* ``reference``: the reference package itself (baseline/_ref, installed from
  /root/reference by __graft_entry__.build(); pkg/src/bimine) --
  ``mine_corpus(model, lexicon, pairs, MiningConfig(workers=W), engine="nw")``
  (align.py:402-448) at W = 1 and W = os.cpu_count() on bounded samples of
  the same documents as text, and DP-only GCUPS of ``kernels.fill_sequential``
  and ``fill_wavefront(workers=W)`` (kernels.py:51-73, the compiled
  ``_nwcore``) on the samples' score matrices;
* ``cpu``: lscpu model name, cores.

Test/measurement infrastructure only: nothing in the package imports it.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def cpu_info() -> dict:
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.lower().startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except (OSError, subprocess.SubprocessError):
        pass
    return {"model": model, "logical_cpus": os.cpu_count()}


def port_rate(corpus, model_vec, seconds: float) -> dict:
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import oracle

    oracle.build()
    threads = oracle.max_threads()
    d = corpus.dictionary
    od = oracle.OracleDict(d.src, d.tgt, d.prob)
    b = corpus.batch
    probe = b.select(range(min(64, b.n_pairs)))
    t0 = time.perf_counter()
    oracle.mine_batch(od, model_vec, probe, threads=threads)
    rate = probe.n_pairs / max(time.perf_counter() - t0, 1e-6)
    n = int(min(b.n_pairs, max(probe.n_pairs, rate * seconds)))
    sample = b.select(range(n))
    t0 = time.perf_counter()
    oracle.mine_batch(od, model_vec, sample, threads=threads)
    dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": "doc_pairs/s", "cores": threads, "kind": "port",
            "sample": f"first {n} of the {b.n_pairs} pairs ({sample.n_cells} cells), oracle/bimine_oracle.c "
                      f"mine_batch with {threads} OpenMP threads, {dt:.1f}s",
            "cells_per_s": sample.n_cells / dt}


def reference_rates(corpus, seconds: float) -> dict:
    ref_dir = os.path.join(REPO, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "bimine")):
        return {"unavailable": "baseline/_ref/bimine not installed (build() installs it from /root/reference)"}
    sys.path.insert(0, ref_dir)
    from bimine import kernels
    from bimine.align import MiningConfig, build_score_matrix, mine_corpus
    from bimine.classifier import load_model
    from bimine.corpus import Document, DocumentPair
    from bimine.lexicon import Lexicon

    model = load_model(os.path.join(REPO, "tests", "golden", "synth_model.json"))
    lexicon = Lexicon(corpus.dictionary.table())
    b = corpus.batch

    def doc_pairs(lo, hi):
        out = []
        for p in range(lo, hi):
            src, tgt = corpus.pair_sentences(p)
            out.append(DocumentPair(topic_id=f"p{p}", source=Document(id=f"s{p}", lang="pl", title=str(p),
                                                                     sentences=tuple(src)),
                                    target=Document(id=f"t{p}", lang="en", title=str(p), sentences=tuple(tgt))))
        return out

    res = {"package": "bimine 0.1.0 (baseline/_ref, compiled _nwcore: %s)" % kernels.backend_name(),
           "path": "mine_corpus(model, lexicon, pairs, MiningConfig(workers=W), engine='nw') -- align.py:402-448"}
    workers_all = os.cpu_count() or 1
    for w in sorted({1, workers_all}):
        # calibrate on 4 pairs per worker, then size the sample to ~seconds
        probe = doc_pairs(0, min(b.n_pairs, 4 * w))
        t0 = time.perf_counter()
        mine_corpus(model, lexicon, probe, MiningConfig(workers=w), engine="nw")
        rate = len(probe) / max(time.perf_counter() - t0, 1e-6)
        n = int(min(b.n_pairs, max(len(probe), rate * seconds / 2)))
        sample = doc_pairs(0, n)
        t0 = time.perf_counter()
        out = mine_corpus(model, lexicon, sample, MiningConfig(workers=w), engine="nw")
        dt = time.perf_counter() - t0
        cells = int(np.sum(b.pair_n[:n].astype(np.int64) * b.pair_m[:n]))
        res[f"workers_{w}"] = {"pairs_per_s": n / dt, "pairs": n, "seconds": dt, "rows": len(out.rows),
                               "failures": len(out.failures), "cells_per_s": cells / dt}
    # DP only: the compiled fill on the first pairs' score matrices
    sims = []
    for p in range(min(b.n_pairs, 40)):
        src, tgt = corpus.pair_sentences(p)
        sims.append(build_score_matrix(model, lexicon, src, tgt)[::-1, ::-1].copy())
    cells = sum(s.size for s in sims)
    reps = 0
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < min(3.0, seconds / 4) or reps == 0:
        for s in sims:
            kernels.fill_sequential(s, -1.0, 1.0, 2.0)
        reps += 1
    seq = cells * reps / (time.perf_counter() - t0) / 1e9
    reps = 0
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < min(3.0, seconds / 4) or reps == 0:
        for s in sims:
            kernels.fill_wavefront(s, -1.0, 1.0, 2.0, workers_all)
        reps += 1
    wav = cells * reps / (time.perf_counter() - t0) / 1e9
    res["dp_gcups"] = {"fill_sequential": seq, f"fill_wavefront_workers_{workers_all}": wav,
                       "sample": f"{len(sims)} score matrices of the workload ({cells} cells), reversed as "
                                 "align.py:166-179 passes them"}
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--pairs", type=int, default=None)
    ap.add_argument("--seconds", type=float, default=15.0)
    ap.add_argument("--port-only", action="store_true")
    args = ap.parse_args()
    from bench import load_workload

    corpus, model_vec = load_workload(args.config, args.pairs, 0)
    out = {"cpu": cpu_info(), "port": port_rate(corpus, model_vec, args.seconds)}
    if not args.port_only:
        out["reference"] = reference_rates(corpus, args.seconds)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
