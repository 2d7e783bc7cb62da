"""bench.py's launch and sharding logic (CPU).

* `--gpus N` outside torchrun re-launches under torch.distributed.run only
  when N GPUs are visible; otherwise it exits non-zero with the reason
  (never a silent one-GPU run labelled as N).
* Under torchrun the world size must equal --gpus.
* C5's 1,000,000 descriptors split into contiguous, cell-balanced rank
  shares that tile [0, total) exactly, each a valid batch over the base
  sentences.
"""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import bench  # noqa: E402


def _visible_gpus():
    try:
        import torch

        return torch.cuda.device_count() if torch.cuda.is_available() else 0
    except Exception:
        return 0


def test_gpus_beyond_visible_exits_nonzero():
    n = max(2, _visible_gpus() + 1)
    res = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", str(n), "--steps", "1",
                          "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=REPO)
    assert res.returncode != 0
    line = json.loads([x for x in res.stdout.splitlines() if x.startswith("{")][-1])
    assert "error" in line and f"--gpus {n}" in line["error"]
    assert "value" not in line


def test_world_size_must_match_gpus():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    res = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "4", "--steps", "1"],
                         capture_output=True, text=True, timeout=600, cwd=REPO, env=env)
    assert res.returncode == 2
    assert "WORLD_SIZE=2" in res.stderr


@pytest.fixture(scope="module")
def base():
    corpus, _ = bench.load_workload(2, 300, 0)
    return corpus.batch


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_c5_shards_tile_the_descriptors(base, world):
    total = 20_000
    idx, cells = bench.c5_descriptors(base, total)
    shards = [bench.c5_shard(base, total, r, world) for r in range(world)]
    assert shards[0][1] == 0 and shards[-1][2] == total
    for (b, lo, hi), nxt in zip(shards, shards[1:] + [(None, total, None)]):
        assert hi == nxt[1]
        # the shard's descriptors are base pairs idx[lo:hi], simulation offsets packed from 0
        assert np.array_equal(b.pair_n, base.pair_n[idx[lo:hi]])
        assert np.array_equal(b.pair_src, base.pair_src[idx[lo:hi]])
        assert b.n_cells == int(cells[lo:hi].sum())
        assert b.tokens is base.tokens  # sentences shared, not copied
    per = np.array([s[0].n_cells for s in shards], dtype=np.float64)
    assert per.max() / per.mean() < 1.01  # balanced by N*M


def test_c5_default_total_is_one_million():
    assert bench.C5_TOTAL == 1_000_000
