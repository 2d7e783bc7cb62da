"""TEST INFRASTRUCTURE ONLY: ctypes bindings of the CPU oracle.

Importable by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs, never by the product package.
Wraps ``liboracle_bimine.so`` (bimine_oracle.c, the plain-C restatement
of the reference path) and ``_ref/_nwcore*.so`` (the reference's own
compiled fill kernels, when built).
"""

from __future__ import annotations

import ctypes
import glob
import math
import importlib.util
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle_bimine.so")

_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)
_f64p = ctypes.POINTER(ctypes.c_double)
_u8p = ctypes.POINTER(ctypes.c_uint8)


class CBatch(ctypes.Structure):
    _fields_ = [
        ("n_pairs", ctypes.c_int64),
        ("n_sentences", ctypes.c_int64),
        ("n_tokens", ctypes.c_int64),
        ("tokens", _i32p),
        ("sent_tok_off", _i64p),
        ("sent_len", _i32p),
        ("sent_uniq", _i32p),
        ("sent_chars", _i32p),
        ("pair_src", _i64p),
        ("pair_n", _i32p),
        ("pair_tgt", _i64p),
        ("pair_m", _i32p),
        ("pair_sim_off", _i64p),
    ]


class CDictView(ctypes.Structure):
    _fields_ = [
        ("n_rows", ctypes.c_int64),
        ("n_entries", ctypes.c_int64),
        ("row_ptr", _i64p),
        ("tgt", _i32p),
        ("prob", _f64p),
    ]


class CMatch(ctypes.Structure):
    _fields_ = [("score", ctypes.c_double), ("i", ctypes.c_int32), ("j", ctypes.c_int32)]


MATCH_DTYPE = np.dtype([("score", "<f8"), ("i", "<i4"), ("j", "<i4")])


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def build() -> str:
    """Compile the oracle (and oracle/_ref when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True, stdout=sys.stderr)  # keep stdout for JSON lines
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        L.oracle_score_batch.argtypes = [ctypes.POINTER(CDictView), _f64p, ctypes.POINTER(CBatch), _f64p, ctypes.c_int]
        L.oracle_mine_batch.argtypes = [
            ctypes.POINTER(CDictView), _f64p, ctypes.POINTER(CBatch), ctypes.c_double, ctypes.c_double,
            ctypes.c_double, ctypes.c_double, _i64p, ctypes.POINTER(CMatch), _i32p, ctypes.c_int,
        ]
        L.oracle_nw_align.argtypes = [_f64p, ctypes.c_int64, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                                      ctypes.c_double, _u8p, _i32p, _i32p, _f64p]
        L.oracle_nw_align.restype = ctypes.c_int64
        L.oracle_nw_fill.argtypes = [_f64p, _f64p, ctypes.c_int64, ctypes.c_int64, ctypes.c_double, ctypes.c_double, ctypes.c_double]
        L.oracle_init_table.argtypes = [_f64p, ctypes.c_int64, ctypes.c_int64, ctypes.c_double]
        L.oracle_exp_array.argtypes = [_f64p, _f64p, ctypes.c_int64]
        L.oracle_max_threads.restype = ctypes.c_int
        _lib = L
    return _lib


class OracleDict:
    """CSR of a lexicon's (src, tgt, p) COO arrays: p > 0 only, a repeated
    (src, tgt) keeps its last value (read_lexicon, lexicon.py:177)."""

    def __init__(self, src, tgt, prob):
        src = np.asarray(src, dtype=np.int64)
        tgt = np.asarray(tgt, dtype=np.int64)
        prob = np.asarray(prob, dtype=np.float64)
        if src.size:
            key = src << 32 | (tgt & 0xFFFFFFFF)
            _, last_rev = np.unique(key[::-1], return_index=True)
            keep = np.sort(src.size - 1 - last_rev)
            src, tgt, prob = src[keep], tgt[keep], prob[keep]
            pos = prob > 0.0
            src, tgt, prob = src[pos], tgt[pos], prob[pos]
        order = np.argsort(src, kind="stable")
        n_rows = int(src.max()) + 1 if src.size else 0
        self.row_ptr = np.zeros(n_rows + 1, dtype=np.int64)
        if src.size:
            np.cumsum(np.bincount(src, minlength=n_rows), out=self.row_ptr[1:])
        self.tgt = np.ascontiguousarray(tgt[order], dtype=np.int32)
        self.prob = np.ascontiguousarray(prob[order], dtype=np.float64)
        self.view = CDictView(n_rows, self.tgt.size, _ptr(self.row_ptr, _i64p), _ptr(self.tgt, _i32p), _ptr(self.prob, _f64p))


def batch_struct(b) -> CBatch:
    return CBatch(
        b.n_pairs, b.n_sentences, b.n_tokens,
        _ptr(b.tokens, _i32p), _ptr(b.sent_tok_off, _i64p), _ptr(b.sent_len, _i32p),
        _ptr(b.sent_uniq, _i32p), _ptr(b.sent_chars, _i32p), _ptr(b.pair_src, _i64p),
        _ptr(b.pair_n, _i32p), _ptr(b.pair_tgt, _i64p), _ptr(b.pair_m, _i32p),
        _ptr(b.pair_sim_off, _i64p),
    )


def score_batch(d: OracleDict, model_vec: np.ndarray, batch, threads: int = 0) -> np.ndarray:
    """build_score_matrix for every pair; flat array at pair_sim_off."""
    sim = np.empty(max(batch.n_cells, 1), dtype=np.float64)
    cb = batch_struct(batch)
    mv = np.ascontiguousarray(model_vec, dtype=np.float64)
    lib().oracle_score_batch(ctypes.byref(d.view), _ptr(mv, _f64p), ctypes.byref(cb), _ptr(sim, _f64p), threads)
    return sim[: batch.n_cells]


def mine_batch(d: OracleDict, model_vec, batch, gap=2.0, threshold=0.5, mismatch=-1.0, bonus=1.0, threads: int = 0):
    """align_pair_indices for every pair -> (counts[P], list of match arrays)."""
    off = batch.match_capacity()
    out = np.zeros(max(int(off[-1]), 1), dtype=MATCH_DTYPE)
    counts = np.zeros(batch.n_pairs, dtype=np.int32)
    cb = batch_struct(batch)
    mv = np.ascontiguousarray(model_vec, dtype=np.float64)
    lib().oracle_mine_batch(
        ctypes.byref(d.view), _ptr(mv, _f64p), ctypes.byref(cb), gap, threshold, mismatch, bonus,
        _ptr(off, _i64p), out.ctypes.data_as(ctypes.POINTER(CMatch)), _ptr(counts, _i32p), threads,
    )
    return counts, [out[off[p] : off[p] + counts[p]] for p in range(batch.n_pairs)]


def nw_align(sim: np.ndarray, mismatch: float, bonus: float, gap: float):
    """nw_align (align.py:170-181) -> (codes uint8[k], i int32[k], j int32[k], score)."""
    sim = np.ascontiguousarray(sim, dtype=np.float64)
    n, m = sim.shape
    steps = np.zeros(n + m, dtype=np.uint8)
    si = np.zeros(n + m, dtype=np.int32)
    sj = np.zeros(n + m, dtype=np.int32)
    score = ctypes.c_double()
    k = lib().oracle_nw_align(_ptr(sim, _f64p), n, m, mismatch, bonus, gap, _ptr(steps, _u8p), _ptr(si, _i32p), _ptr(sj, _i32p), ctypes.byref(score))
    return steps[:k], si[:k], sj[:k], score.value


def nw_table(rev_sim: np.ndarray, mismatch: float, bonus: float, gap: float) -> np.ndarray:
    """kernels.fill_sequential (kernels.py:51-58) on an already reversed matrix."""
    rev_sim = np.ascontiguousarray(rev_sim, dtype=np.float64)
    n, m = rev_sim.shape
    dp = np.empty((n + 1, m + 1), dtype=np.float64)
    lib().oracle_init_table(_ptr(dp, _f64p), n, m, gap)
    lib().oracle_nw_fill(_ptr(dp, _f64p), _ptr(rev_sim, _f64p), n, m, mismatch, bonus, gap)
    return dp


def exp_array(x: np.ndarray) -> np.ndarray:
    """libm exp -- the function CPython's math.exp calls."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty_like(x)
    lib().oracle_exp_array(_ptr(x, _f64p), _ptr(y, _f64p), x.size)
    return y


def max_threads() -> int:
    return int(lib().oracle_max_threads())


def reference_nwcore():
    """The reference's own compiled _nwcore module from oracle/_ref, or None."""
    paths = glob.glob(os.path.join(HERE, "_ref", "_nwcore*.so"))
    if not paths:
        return None
    spec = importlib.util.spec_from_file_location("_nwcore", paths[0])
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


# ---------------------------------------------------------------------------
# f4: lexicon EM, restated in plain Python (lexicon.py:60-120).  Test
# infrastructure only: the product runs the rounds on the GPU.
# ---------------------------------------------------------------------------

def py_sum(values):
    """CPython >= 3.12 built-in sum() over floats (Python/bltinmodule.c):
    0 + x0, then Neumaier's compensated steps, the compensation added at the
    end when it is nonzero and finite -- what `sum(row_counts.values())`
    computes in lexicon.py:112."""
    it = iter(values)
    try:
        f = 0 + next(it)
    except StopIteration:
        return 0
    c = 0.0
    for x in it:
        t = f + x
        if abs(f) >= abs(x):
            c = c + ((f - t) + x)
        else:
            c = c + ((x - t) + f)
        f = t
    if c and math.isfinite(c):
        f = f + c
    return f


def build_lexicon(parallel, iterations, prune_threshold=1e-4, tokenize=None):
    """dict[s][t] -> p with the reference's float64 operation order: per
    round, for every pair in order and every source occurrence in order,
    denom = sequential sum over the target positions; counts[s][t] += p/denom
    per position; rows renormalised by Python's sum() (compensated, see
    py_sum) of their counts in first-count order."""
    if tokenize is None:
        sys.path.insert(0, os.path.dirname(HERE))
        from paper_1512_01641_b200.text import tokenize
    if not parallel:
        raise ValueError("no training pairs")
    if iterations < 1:
        raise ValueError("iterations must be >= 1")
    data = [(a, b) for a, b in ((tokenize(x), tokenize(y)) for x, y in parallel) if a and b]
    if not data:
        raise ValueError("no training pairs")
    support = {}
    for src, tgt in data:
        for s in src:
            support.setdefault(s, set()).update(tgt)
    prob = {s: dict.fromkeys(ts, 1.0 / len(ts)) for s, ts in support.items()}
    for _ in range(iterations):
        counts = {s: {} for s in prob}
        for src, tgt in data:
            for s in src:
                row = prob[s]
                denom = 0.0
                for t in tgt:
                    denom = denom + row[t]
                if not denom > 0.0:
                    continue
                acc = counts[s]
                for t in tgt:
                    acc[t] = acc.get(t, 0.0) + row[t] / denom
        for s, acc in counts.items():
            total = py_sum(acc.values())  # first-count (insertion) order
            if total > 0.0:
                prob[s] = {t: v / total for t, v in acc.items()}
    if prune_threshold > 0.0:
        kept = {s: {t: p for t, p in row.items() if p >= prune_threshold} for s, row in prob.items()}
        prob = {s: row for s, row in kept.items() if row}
    return prob
