"""bimine_mine_host's host/device timeline on C2 (run against a build with
-DBIMINE_E2E_PROFILE, e.g. BIMINE_LIB=scratch_so/e2eprof.so): prints the
library's per-call timeline line for a few calls: the compact wire form
(24-bit ids, uint16 sentence arrays), 24-bit ids only, int32.

    BIMINE_LIB=scratch_so/e2eprof.so python tools/e2e_timeline.py
"""
import sys

sys.path[:0] = ["."]
import numpy as np
import torch

import bench
from paper_1512_01641_b200 import engine as E

corpus, model = bench.load_workload(2, 10000, 0)
d = corpus.dictionary
dd = E.LexiconContext(vocab=None, coo=(d.src, d.tgt, d.prob), devices={}).on(0)


class _R:
    pass


R = _R()
R.torch = torch
for name, b in (("wire", corpus.batch.with_24bit_tokens().with_narrow_sentences()),
                ("24-bit", corpus.batch.with_24bit_tokens()), ("int32", corpus.batch)):
    pb = bench.pinned_batch(R, b)
    out = {}
    for k in range(5):
        sys.stderr.write(f"[{name} call {k}] ")
        sys.stderr.flush()
        E.mine_host(dd, model, pb, 2.0, 0.5, -1.0, 1.0, out=out)
        torch.cuda.synchronize()
