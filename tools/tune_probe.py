"""Phase timing of engine.tune_device on C4 (1k pairs x 64 settings)."""
import sys
import time

sys.path[:0] = ["."]
import numpy as np
import torch

import bench
from paper_1512_01641_b200 import engine as E

corpus, model = bench.load_workload(4, None, 0)
thr, gaps, refs = bench._tuning_inputs(corpus)
d = corpus.dictionary
dd = E.LexiconContext(vocab=None, coo=(d.src, d.tgt, d.prob), devices={}).on(0)
b = corpus.batch
for _ in range(2):
    E.tune_device(dd, model, b, thr, gaps, -1.0, 1.0, refs)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    E.tune_device(dd, model, b, thr, gaps, -1.0, 1.0, refs)
print(f"tune_device {(time.perf_counter() - t) / 5 * 1e3:.2f} ms")
t = time.perf_counter()
for _ in range(5):
    db = E.DeviceBatch(b, 0)
torch.cuda.synchronize()
print(f"DeviceBatch {(time.perf_counter() - t) / 5 * 1e3:.2f} ms")
t = time.perf_counter()
for _ in range(5):
    flat = [np.asarray(r, dtype=np.int32).reshape(-1) for r in refs if len(r)]
    np.concatenate(flat)
print(f"refs flatten {(time.perf_counter() - t) / 5 * 1e3:.2f} ms")
