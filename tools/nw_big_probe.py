"""Run the band-pipeline NW on one shape and check it against the oracle."""
import sys
import time

sys.path[:0] = [".", "oracle", "tests"]
import numpy as np
import oracle
from paper_1512_01641_b200 import engine as E

n, m = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(1)
sim = rng.random((n, m))
t = time.time()
[(codes, score)] = E.nw_steps_host([sim], [1.3], -1.0, 1.0)
dt = time.time() - t
want, _, _, ws = oracle.nw_align(sim, -1.0, 1.0, 1.3)
print(n, m, "ok" if np.array_equal(codes, want) and score == ws else "MISMATCH", f"{dt:.3f}s", flush=True)
