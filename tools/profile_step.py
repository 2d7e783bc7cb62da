"""One mining step on a synthetic batch, for ncu captures.

    python tools/profile_step.py [--config 2] [--pairs 2000] [--repeat 2]

Runs score kernel -> NW/traceback/filter -> compaction `repeat` times on a
device-resident batch (first pass = warm-up), nothing else.
"""

import argparse
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--pairs", type=int, default=2000)
    ap.add_argument("--repeat", type=int, default=2)
    args = ap.parse_args()
    import torch

    from bench import load_workload
    from paper_1512_01641_b200 import engine as E

    corpus, model = load_workload(args.config, args.pairs, 0)
    d = corpus.dictionary
    ctx = E.LexiconContext(vocab=None, coo=(d.src, d.tgt, d.prob), devices={})
    dd = ctx.on(0)
    db = E.DeviceBatch(corpus.batch, 0)
    sim = torch.empty(max(corpus.batch.n_cells, 1), dtype=torch.float64, device="cuda:0")
    out = None
    for _ in range(args.repeat):
        out = E.mine_device(dd, model, db, sim, 2.0, 0.5, -1.0, 1.0, out=out)
    torch.cuda.synchronize()
    print("matches", int(out["total"].item()), "cells", corpus.batch.n_cells)


if __name__ == "__main__":
    main()
