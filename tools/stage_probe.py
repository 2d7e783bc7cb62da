"""Pageable vs pinned bimine_mine_host on C2 (e2e), host memcpy bandwidth.

    python tools/stage_probe.py [threads...]

Runs each setting of BIMINE_STAGE_THREADS in a fresh process (the memcpy
pool is created once per process).
"""
import json
import os
import subprocess
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

CHILD = r'''
import sys, time, json, numpy as np
sys.path.insert(0, sys.argv[1])
import torch, bench
from paper_1512_01641_b200 import engine as E
corpus, model = bench.load_workload(2, None, 0)
b = corpus.batch; d = corpus.dictionary
dd = E.LexiconContext(vocab=None, coo=(d.src, d.tgt, d.prob), devices={}).on(0)
out = {}
res = {}
for kind in ("pageable", "pinned"):
    bb = b
    if kind == "pinned":
        from paper_1512_01641_b200.packing import PackedBatch
        bb = PackedBatch(**{f: torch.from_numpy(np.ascontiguousarray(getattr(b, f))).pin_memory().numpy()
                            for f in ("tokens","sent_tok_off","sent_len","sent_uniq","sent_chars","pair_src","pair_n","pair_tgt","pair_m","pair_sim_off")})
    for _ in range(3):
        E.mine_host(dd, model, bb, 2.0, 0.5, -1.0, 1.0, out=out)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(20):
        E.mine_host(dd, model, bb, 2.0, 0.5, -1.0, 1.0, out=out)
    res[kind] = (time.perf_counter() - t) / 20 * 1e3
# host memcpy bandwidth (one thread)
src = np.ones(100_000_000 // 8); dst = np.empty_like(src)
t = time.perf_counter(); np.copyto(dst, src); res["memcpy_1thread_GBps"] = 0.8 / (time.perf_counter() - t)
print(json.dumps(res))
'''


def main():
    settings = sys.argv[1:] or ["1", "3", "5", "7", "11"]
    for th in settings:
        env = dict(os.environ, BIMINE_STAGE_THREADS=th)
        r = subprocess.run([sys.executable, "-c", CHILD, REPO], capture_output=True, text=True, env=env)
        line = [x for x in r.stdout.splitlines() if x.startswith("{")]
        print(th, line[-1] if line else r.stderr[-1500:], flush=True)


if __name__ == "__main__":
    main()
