"""Raw H2D bandwidth on the box vs bimine_mine_host's upload pattern
(16 pieces, a 4-byte counter copy after each).  CUDA events, pinned source.
    python tools/h2d_probe.py [MB]
"""
import sys

import torch

mb = float(sys.argv[1]) if len(sys.argv) > 1 else 79.0
n = int(mb * 1e6)
src = torch.empty(n, dtype=torch.uint8, pin_memory=True)
src.fill_(1)
dst = torch.empty(n, dtype=torch.uint8, device="cuda")
ctr_h = torch.arange(64, dtype=torch.int32).pin_memory()
ctr_d = torch.zeros(1, dtype=torch.int32, device="cuda")
s = torch.cuda.Stream()


def run(pieces, bumps):
    with torch.cuda.stream(s):
        cut = [n * k // pieces for k in range(pieces + 1)]
        for k in range(pieces):
            dst[cut[k]:cut[k + 1]].copy_(src[cut[k]:cut[k + 1]], non_blocking=True)
            if bumps:
                ctr_d.copy_(ctr_h[k:k + 1], non_blocking=True)


for pieces, bumps in ((1, False), (4, False), (16, False), (16, True), (64, True)):
    for _ in range(3):
        run(pieces, bumps)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(10):
        e0.record(s)
        run(pieces, bumps)
        e1.record(s)
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"{pieces:3d} pieces bumps={bumps}: {best:.3f} ms = {n / best / 1e6:.1f} GB/s")
