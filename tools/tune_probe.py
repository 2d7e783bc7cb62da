"""Per-call and per-phase timing of engine.tune_device on C4 (1k pairs x 64
settings) with a persistent DeviceTuner; device phases by CUDA events.

    python tools/tune_probe.py [calls]
"""
import sys
import time

sys.path[:0] = ["."]
import numpy as np
import torch

import bench
from paper_1512_01641_b200 import engine as E

calls = int(sys.argv[1]) if len(sys.argv) > 1 else 30
corpus, model = bench.load_workload(4, None, 0)
thr, gaps, refs = bench._tuning_inputs(corpus)
d = corpus.dictionary
dd = E.LexiconContext(vocab=None, coo=(d.src, d.tgt, d.prob), devices={}).on(0)
b = corpus.batch
tuner = E.DeviceTuner(dd, model, b, thr, gaps, -1.0, 1.0, refs)
for _ in range(3):
    E.tune_device(dd, model, b, thr, gaps, -1.0, 1.0, refs, tuner=tuner)
torch.cuda.synchronize()
walls, up, dev, res = [], [], [], []
for _ in range(calls):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    t0 = time.perf_counter()
    tuner.upload(b)
    t1 = time.perf_counter()
    tuner.run_device(events=ev)
    t2 = time.perf_counter()
    tuner.results()
    t3 = time.perf_counter()
    walls.append(t3 - t0)
    up.append(t1 - t0)
    res.append(t3 - t2)
    dev.append([ev[i].elapsed_time(ev[i + 1]) for i in range(3)])
walls = np.array(walls) * 1e3
dev = np.array(dev)
print(f"call ms: min {walls.min():.2f} median {np.median(walls):.2f} max {walls.max():.2f}")
print(f"host upload ms median {np.median(up) * 1e3:.2f}; results wait ms median {np.median(res) * 1e3:.2f}")
print("device ms (score, nw, agreement): median", np.median(dev, axis=0).round(3), "min", dev.min(axis=0).round(3),
      "max", dev.max(axis=0).round(3))
t = time.perf_counter()
for _ in range(calls):
    E.tune_device(dd, model, b, thr, gaps, -1.0, 1.0, refs, tuner=tuner)
print(f"tune_device loop: {(time.perf_counter() - t) / calls * 1e3:.2f} ms/call = {b.n_pairs * calls / (time.perf_counter() - t):.0f} pairs/s")
