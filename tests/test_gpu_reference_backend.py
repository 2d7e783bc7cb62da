"""The reference package itself, with the B200 fill registered as a backend.

baseline/_ref holds the reference (pkg/src/bimine, compiled _nwcore),
installed from /root/reference by __graft_entry__.build().  Registering
paper_1512_01641_b200.nwcore_cuda as bimine.kernels._BACKENDS["cuda"]
(kernels.py:29-31; no reference file changed), the reference's own checks
run against it:

* test_backends_produce_identical_tables (pkg/tests/test_align.py:152-166):
  every backend's fill_sequential / fill_wavefront table np.array_equal;
* criterion 2's instance family (pkg/tests/test_acceptance.py:89-110: 500
  random instances up to 200x200, seed 2002): nw_align and
  nw_align_wavefront with backend="cuda" equal to the compiled backend's
  (score and step list).
"""

import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU containers
    pytest.skip("needs a CUDA device", allow_module_level=True)

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(REPO, "baseline", "_ref")
if not os.path.isdir(os.path.join(REF, "bimine")):  # pragma: no cover
    pytest.skip("baseline/_ref (the reference package) not installed", allow_module_level=True)
sys.path.insert(0, REF)

from bimine import kernels  # noqa: E402
from bimine.align import MiningConfig, nw_align, nw_align_wavefront  # noqa: E402

from paper_1512_01641_b200 import nwcore_cuda  # noqa: E402

nwcore_cuda.register(kernels)


def test_cuda_backend_registered():
    assert "cuda" in kernels.available_backends()
    assert kernels._BACKENDS["cuda"] is nwcore_cuda
    assert kernels.backend_name() == "compiled"  # the reference's own default is untouched


def test_backends_produce_identical_tables():
    rng = np.random.default_rng(31)
    available = kernels.available_backends()
    assert {"python", "compiled", "cuda"} <= set(available)
    for _ in range(10):
        sim = rng.random((int(rng.integers(1, 60)), int(rng.integers(1, 60))))
        tables = [kernels.fill_sequential(sim, -1.0, 1.0, 0.7, backend=b) for b in available]
        assert all(np.array_equal(tables[0], t) for t in tables[1:])
        waves = [kernels.fill_wavefront(sim, -1.0, 1.0, 0.7, 3, backend=b) for b in available]
        assert all(np.array_equal(tables[0], w) for w in waves)


def test_acceptance_family_through_the_reference_api():
    rng = np.random.default_rng(2002)
    for _ in range(500):
        n = int(rng.integers(1, 201))
        m = int(rng.integers(1, 201))
        sim = rng.random((n, m))
        config = MiningConfig(gap_penalty=float(rng.uniform(0.0, 3.0)))
        want = nw_align(sim, config, backend="compiled")
        got = nw_align(sim, config, backend="cuda")
        assert got.score == want.score and got.steps == want.steps
        wave = nw_align_wavefront(sim, config, 4, backend="cuda")
        assert wave == want


def test_buffer_contract_errors():
    sim = np.random.default_rng(1).random((5, 7))
    with pytest.raises(ValueError):
        nwcore_cuda.nw_fill(np.zeros((6, 8), dtype=np.float32), sim, -1.0, 1.0, 1.0)
    with pytest.raises(ValueError):
        nwcore_cuda.nw_fill(np.zeros((5, 8)), sim, -1.0, 1.0, 1.0)
    with pytest.raises(ValueError):
        nwcore_cuda.nw_fill_wavefront(np.zeros((6, 8)), sim, -1.0, 1.0, 1.0, 0)
