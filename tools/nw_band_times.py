"""Band end times of one 4096x4096 cluster sweep from a -DBIMINE_PROF_GLOBAL
build (globaltimer stamps in a device array: no printf call site in the
kernel).    BIMINE_LIB=scratch_so/X.so python tools/nw_band_times.py [n m]
"""
import ctypes
import statistics
import sys

sys.path[:0] = ["."]
import numpy as np

from paper_1512_01641_b200 import _native as N
from paper_1512_01641_b200 import engine as E

n, m = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (4096, 4096)
sim = np.random.default_rng(1).random((n, m))
E.nw_steps_host([sim], [1.3], -1.0, 1.0)
E.nw_steps_host([sim], [1.3], -1.0, 1.0)
L = N.load()
t = np.zeros(4096, np.uint64)
L.bimine_debug_band_times.argtypes = [ctypes.c_void_p, ctypes.c_int]
assert L.bimine_debug_band_times(t.ctypes.data, 4096) == 0
G = (n + 31) // 32
e = t[:G].astype(np.int64)
t0 = int(t[4095])
print(f"band 0: {(e[0] - t0) / 1e3:.1f} us = {(e[0] - t0) / (m + 31) * 1.965:.0f} cycles per step; last band end {(e[-1] - t0) / 1e3:.1f} us")
lag = np.diff(e) / 1e3
print(f"band0 end->last end: {(e[-1] - e[0]) / 1e3:.1f} us over {G - 1} lags; lag median {statistics.median(lag):.2f} us")
print("lag by warp:", [round(statistics.median(lag[w::8]), 2) for w in range(8)])
print("first lags:", np.round(lag[:12], 1).tolist())
