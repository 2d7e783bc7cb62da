"""Timing guard for the cluster NW sweep's codegen sensitivity.

nw_big_kernel keeps an unreachable printf call site in its band loop: with
it the 4096x4096 NW (operand layout + sweep + traceback) takes ~2.9 ms,
without it ~5.9 ms -- each band's hand-off lag triples
(profiles/r2/nw_big_printf_ab.txt).  A toolchain change that loses the
effect fails here instead of silently slowing C3.
"""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU containers
    pytest.skip("needs a CUDA device", allow_module_level=True)

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIMIT_MS = 4.0


def test_c3_nw_sweep_keeps_its_schedule():
    r = subprocess.run([sys.executable, os.path.join(REPO, "tools", "nw_time.py"), "4096", "4096", "7"],
                       capture_output=True, text=True, timeout=600, cwd=REPO)
    assert r.returncode == 0, r.stderr[-2000:]
    ms = float(r.stdout.split()[2])
    assert ms < LIMIT_MS, f"4096x4096 NW took {ms:.3f} ms (guard {LIMIT_MS} ms): the band pipeline's schedule regressed"
