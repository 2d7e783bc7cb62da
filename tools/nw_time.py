"""Time the standalone NW (+traceback/filter) of one n x m problem on the
device: python tools/nw_time.py n m [reps].  Prints ms per launch."""
import sys

sys.path[:0] = ["."]
import numpy as np
import torch

from paper_1512_01641_b200 import _native as N

L = N.load()
n, m = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
dev = "cuda:0"
sim = torch.rand(n * m, dtype=torch.float64, device=dev)
i64 = lambda v: torch.tensor(v, dtype=torch.int64, device=dev)
i32 = lambda v: torch.tensor(v, dtype=torch.int32, device=dev)
off, pn, pm = i64([0]), i32([n]), i32([m])
par = torch.tensor([1.3, 0.5], dtype=torch.float64, device=dev)
out_off = i64([0, min(n, m)])
slots = torch.empty(min(n, m) * 16, dtype=torch.uint8, device=dev)
counts = torch.zeros(1, dtype=torch.int32, device=dev)
st = torch.cuda.current_stream().cuda_stream


def run():
    N.check(L.bimine_nw_mine_batch(sim.data_ptr(), off.data_ptr(), pn.data_ptr(), pm.data_ptr(), 1, n, m, 1,
                                   par.data_ptr(), par.data_ptr() + 8, -1.0, 1.0, out_off.data_ptr(),
                                   slots.data_ptr(), counts.data_ptr(), None, st))


run()
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    run()
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
t = min(ts)
print(f"{n} {m} {t:.3f} ms  {n * m / t / 1e6:.3f} GCUPS  {t / ((n + 31) // 32) * 1e3:.1f} us/band", flush=True)
