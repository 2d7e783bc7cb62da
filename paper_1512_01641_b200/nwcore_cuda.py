"""The reference's native kernel plugin, on the B200: a module with the
`_nwcore` surface (pkg/src/bimine/_nwcore.pyx:19-36, 45-70) that the
reference selects through its backend registry (kernels.py:29-31, 51-73).

    from paper_1512_01641_b200 import nwcore_cuda
    nwcore_cuda.register()            # bimine.kernels._BACKENDS["cuda"] = this module
    bimine.align.nw_align(scores, config, backend="cuda")

Same contract as the Cython functions: `dp` is the caller-allocated,
writable C-contiguous float64 (n+1) x (m+1) table with row 0 / column 0
initialised (kernels.py:42-48), `sim` the already reversed n x m score
matrix (kernels.py:55,70); the interior is written in place with values
bit-identical to the reference fill.  `workers` is accepted for signature
compatibility (the anti-diagonal split is the GPU's).  Buffer mismatches
raise ValueError like the Cython memoryview checks would raise their
errors; a device failure raises BimineError.  No CPU fallback.
"""

from __future__ import annotations

import numpy as np

from . import _native as N


def _check_buffers(dp, sim):
    if not isinstance(dp, np.ndarray) or dp.dtype != np.float64 or dp.ndim != 2:
        raise ValueError("dp must be a 2-D float64 array")
    if not dp.flags.c_contiguous or not dp.flags.writeable:
        raise ValueError("dp must be a writable C-contiguous array (double[:, ::1])")
    if not isinstance(sim, np.ndarray) or sim.dtype != np.float64 or sim.ndim != 2 or not sim.flags.c_contiguous:
        raise ValueError("sim must be a C-contiguous 2-D float64 array (const double[:, ::1])")
    n, m = sim.shape
    if dp.shape != (n + 1, m + 1):
        raise ValueError("dp must have shape (n + 1, m + 1) for an n x m sim")
    return n, m


def nw_fill(dp, sim, mismatch, bonus, gap) -> None:
    """_nwcore.nw_fill (_nwcore.pyx:19-36)."""
    n, m = _check_buffers(dp, sim)
    if n == 0 or m == 0:
        return
    L = N.load()
    N.check(L.bimine_nw_fill(N.ptr(dp, N._f64p), N.ptr(sim, N._f64p), n, m, float(mismatch), float(bonus),
                             float(gap), None))


def nw_fill_wavefront(dp, sim, mismatch, bonus, gap, workers) -> None:
    """_nwcore.nw_fill_wavefront (_nwcore.pyx:45-70)."""
    n, m = _check_buffers(dp, sim)
    if int(workers) < 1:
        raise ValueError("workers must be >= 1")
    if n == 0 or m == 0:
        return
    L = N.load()
    N.check(L.bimine_nw_fill_wavefront(N.ptr(dp, N._f64p), N.ptr(sim, N._f64p), n, m, float(mismatch),
                                       float(bonus), float(gap), int(workers), None))


def register(kernels_module=None, name: str = "cuda") -> None:
    """Add this module to the reference's backend registry (no reference
    file is changed): bimine.kernels._BACKENDS[name] = nwcore_cuda."""
    if kernels_module is None:
        from bimine import kernels as kernels_module  # the reference package on sys.path
    import sys

    kernels_module._BACKENDS[name] = sys.modules[__name__]
