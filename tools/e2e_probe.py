"""Break down one bimine_mine_host call on C2 (host prep vs C call)."""
import sys
import time

sys.path[:0] = ["."]
import numpy as np
import torch

from bench import load_workload
from paper_1512_01641_b200 import _native as N
from paper_1512_01641_b200 import engine as E
from paper_1512_01641_b200.classifier import model_vector
from paper_1512_01641_b200.packing import PackedBatch

corpus, model = load_workload(2, 10000, 0)
d = corpus.dictionary
ctx = E.LexiconContext(vocab=None, coo=(d.src, d.tgt, d.prob), devices={})
dd = ctx.on(0)
mv = model_vector(model) if not isinstance(model, np.ndarray) else model
b = corpus.batch
pinned = {f: torch.from_numpy(np.ascontiguousarray(getattr(b, f))).pin_memory().numpy()
          for f in ("tokens", "sent_tok_off", "sent_len", "sent_uniq", "sent_chars", "pair_src", "pair_n",
                    "pair_tgt", "pair_m", "pair_sim_off")}
pb = PackedBatch(**pinned)
for _ in range(2):
    E.mine_host(dd, mv, pb, 2.0, 0.5, -1.0, 1.0)
torch.cuda.synchronize()
L = N.load()
t = time.perf_counter(); cap = int(pb.match_capacity()[-1]); t_cap = time.perf_counter() - t
t = time.perf_counter(); m = np.zeros(cap, dtype=N.MATCH_DTYPE); t_zero = time.perf_counter() - t
t = time.perf_counter(); cb = N.batch_struct_host(pb); t_struct = time.perf_counter() - t
reps = 5
t = time.perf_counter()
for _ in range(reps):
    E.mine_host(dd, mv, pb, 2.0, 0.5, -1.0, 1.0)
t_all = (time.perf_counter() - t) / reps
counts = np.zeros(pb.n_pairs, dtype=np.int32); total = np.zeros(1, dtype=np.int64)
import ctypes
t = time.perf_counter()
for _ in range(reps):
    N.check(L.bimine_mine_host(dd.handle, N.ptr(mv, N._f64p), ctypes.byref(cb), 2.0, 0.5, -1.0, 1.0,
                               N.ptr(counts, N._i32p), m.ctypes.data, cap, N.ptr(total, N._i64p), None, None))
t_c = (time.perf_counter() - t) / reps
print(f"mine_host {t_all*1e3:.2f} ms | C call {t_c*1e3:.2f} ms | capacity {t_cap*1e3:.2f} ms | zeros {t_zero*1e3:.2f} ms | struct {t_struct*1e3:.2f} ms | nbytes {pb.nbytes()/1e6:.1f} MB")
tok = torch.from_numpy(pinned["tokens"])
dst = torch.empty_like(tok, device="cuda:0")
for _ in range(2):
    dst.copy_(tok, non_blocking=True)
torch.cuda.synchronize()
a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5):
    dst.copy_(tok, non_blocking=True)
c.record()
torch.cuda.synchronize()
ms = a.elapsed_time(c) / 5
print(f"pinned H2D {tok.numel()*4/1e6:.1f} MB in {ms:.3f} ms = {tok.numel()*4/ms/1e6:.1f} GB/s")
outbuf = {}
E.mine_host(dd, mv, pb, 2.0, 0.5, -1.0, 1.0, out=outbuf)
t = time.perf_counter()
for _ in range(reps):
    E.mine_host(dd, mv, pb, 2.0, 0.5, -1.0, 1.0, out=outbuf)
print(f"mine_host with reused outputs {(time.perf_counter() - t) / reps * 1e3:.2f} ms")
t = time.perf_counter()
for _ in range(100):
    cb2 = N.batch_struct_host(pb)
print(f"batch_struct_host {(time.perf_counter() - t) / 100 * 1e3:.3f} ms")
