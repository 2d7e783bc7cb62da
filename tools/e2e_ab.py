import sys, time
sys.path[:0] = ["."]
import numpy as np, torch
import bench
from paper_1512_01641_b200 import engine as E
from paper_1512_01641_b200.packing import PackedBatch
corpus, model = bench.load_workload(2, None, 0)
d = corpus.dictionary
dd = E.LexiconContext(vocab=None, coo=(d.src, d.tgt, d.prob), devices={}).on(0)
b = corpus.batch
pb = PackedBatch(**{f: torch.from_numpy(np.ascontiguousarray(getattr(b, f))).pin_memory().numpy() for f in
                   ("tokens", "sent_tok_off", "sent_len", "sent_uniq", "sent_chars", "pair_src", "pair_n", "pair_tgt", "pair_m", "pair_sim_off")})
stream = torch.cuda.current_stream()
for rnd in range(2):
    for reuse in (False, True):
        out = {} if reuse else None
        E.mine_host(dd, model, pb, 2.0, 0.5, -1.0, 1.0, stream=stream, out=out)
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(10):
            E.mine_host(dd, model, pb, 2.0, 0.5, -1.0, 1.0, stream=stream, out=out)
        dt = (time.perf_counter() - t) / 10
        print(f"round {rnd} reuse={reuse}: {dt*1e3:.2f} ms/step = {b.n_pairs/dt/1e6:.2f}M pairs/s", flush=True)
