"""Device execution of the hot path through the C ABI.

Holds the per-lexicon GPU dictionary (joint vocabulary + CSR uploaded
once per device) and the batched calls the public API in ``align`` and
``tuning`` is built on.  PyTorch provides device memory and streams;
all compute is in libbimine_b200.so.
"""

from __future__ import annotations

import ctypes
import itertools
import threading
import weakref
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .packing import PackedBatch, Vocabulary, lexicon_arrays, new_vocabulary


def _torch():
    import torch

    return torch


class DeviceDictionary:
    """A lexicon's joint vocabulary plus its CSR on one CUDA device."""

    def __init__(self, vocab: Vocabulary, src: np.ndarray, tgt: np.ndarray, prob: np.ndarray, device: int):
        self.vocab = vocab
        self.device = device
        L = N.load()
        torch = _torch()
        handle = ctypes.c_void_p()
        with torch.cuda.device(device):
            N.check(L.bimine_dict_create(N.ptr(src, N._i32p), N.ptr(tgt, N._i32p), N.ptr(prob, N._f64p),
                                         int(src.shape[0]), ctypes.byref(handle)))
        self.handle = handle
        self.n_entries = int(L.bimine_dict_entries(handle))

    def __del__(self):
        h = getattr(self, "handle", None)
        lib = getattr(N, "_lib", None) if N is not None else None  # None at interpreter shutdown
        if h and lib is not None:
            try:
                lib.bimine_dict_destroy(h)
            except Exception:
                pass


@dataclass
class LexiconContext:
    vocab: Vocabulary
    coo: tuple  # (src, tgt, prob) ids in lexicon iteration order
    devices: dict  # device index -> DeviceDictionary

    def on(self, device: int) -> DeviceDictionary:
        d = self.devices.get(device)
        if d is None:
            d = DeviceDictionary(self.vocab, *self.coo, device=device)
            self.devices[device] = d
        return d


_contexts: dict[int, tuple] = {}
_ctx_lock = threading.Lock()


def lexicon_context(lexicon) -> LexiconContext:
    """Cached (vocab, COO) for a lexicon object (ours or the reference's)."""
    key = id(lexicon)
    with _ctx_lock:
        hit = _contexts.get(key)
        if hit is not None and hit[0]() is lexicon:
            return hit[1]
        vocab = new_vocabulary()
        coo = lexicon_arrays(lexicon.items(), vocab)
        ctx = LexiconContext(vocab=vocab, coo=coo, devices={})
        try:
            ref = weakref.ref(lexicon)
        except TypeError:  # objects without weakref support: keep them alive
            ref = (lambda obj: (lambda: obj))(lexicon)
        _contexts[key] = (ref, ctx)
        return ctx


def current_device() -> int:
    N.load()  # raises NativeUnavailable without the library or a GPU
    return _torch().cuda.current_device()


# ---------------------------------------------------------------------------
# device-resident batches
# ---------------------------------------------------------------------------

_FIELDS = ("tokens", "sent_tok_off", "sent_len", "sent_uniq", "sent_chars",
           "pair_src", "pair_n", "pair_tgt", "pair_m", "pair_sim_off")


class DeviceBatch:
    """A PackedBatch copied to one device (torch tensors) + its ABI struct."""

    def __init__(self, batch: PackedBatch, device: int, stream=None, pinned: bool = False):
        torch = _torch()
        self.batch = batch
        self.device = device
        self.t = {}
        for f in _FIELDS:
            a = torch.from_numpy(np.ascontiguousarray(getattr(batch, f)))
            if pinned:
                a = a.pin_memory()
            self.t[f] = a.to(f"cuda:{device}", non_blocking=pinned)
        self.struct = N.batch_struct_device(self.t, batch.n_pairs, batch.n_sentences, batch.n_tokens,
                                            batch.token_bytes)
        self.plan, work = plan_batch(batch)
        self.work_host = work  # kept alive: plan.work_host points into it
        self.t["work"] = torch.from_numpy(work).to(f"cuda:{device}")
        self.plan.work = self.t["work"].data_ptr() if work.size else None
        self.plan.work_host = work.ctypes.data if work.size else None
        self.max_n, self.max_m = int(self.plan.max_n), int(self.plan.max_m)
        cap = batch.match_capacity()
        self.capacity = int(cap[-1])
        self.t["out_off"] = torch.from_numpy(cap[:-1].copy()).to(f"cuda:{device}")


def plan_batch(batch: PackedBatch):
    """bimine_plan_batch on the host arrays -> (CPlan, int64 work array)."""
    L = N.load(require_gpu=False)
    n = batch.pair_n.astype(np.int64)
    m = batch.pair_m.astype(np.int64)
    cap = int(3 * batch.n_pairs + 3 * np.sum(((n + 63) // 64) * ((m + 63) // 64)))
    work = np.zeros(max(cap, 1), dtype=np.int64)
    plan = N.CPlan()
    cb = N.batch_struct_host(batch)
    N.check(L.bimine_plan_batch(ctypes.byref(cb), N.ptr(work, N._i64p), cap, ctypes.byref(plan)))
    return plan, work[: int(plan.work_len)].copy()


def stream_ptr(stream=None) -> int:
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def score_device(dd: DeviceDictionary, model_vec: np.ndarray, db: DeviceBatch, sim, stream=None) -> None:
    """build_score_matrix for every pair of a device batch into `sim` (torch f64)."""
    L = N.load()
    mv = np.ascontiguousarray(model_vec, dtype=np.float64)
    N.check(L.bimine_score_batch(dd.handle, N.ptr(mv, N._f64p), ctypes.byref(db.struct), ctypes.byref(db.plan),
                                 sim.data_ptr(), stream_ptr(stream)))


def mine_device(dd: DeviceDictionary, model_vec: np.ndarray, db: DeviceBatch, sim, gap: float, threshold: float,
                mismatch: float, bonus: float, out: dict | None = None, stream=None, events=None) -> dict:
    """The mining step on a device batch (bimine_mine_batch: score kernel,
    then the NW + traceback + filter launch; the NW runs in the score
    kernel's tail only with BIMINE_FUSE_NW=1) + order-preserving
    compaction; returns device tensors (counts, base, compact, total).
    `events` (3 CUDA events) bracket the mining call and the compaction."""
    torch = _torch()
    L = N.load()
    dev = f"cuda:{db.device}"
    P = db.batch.n_pairs
    if out is None:
        out = {
            "slots": torch.empty(max(db.capacity, 1) * 16, dtype=torch.uint8, device=dev),
            "counts": torch.empty(max(P, 1), dtype=torch.int32, device=dev),
            "base": torch.empty(max(P, 1), dtype=torch.int64, device=dev),
            "compact": torch.empty(max(db.capacity, 1) * 16, dtype=torch.uint8, device=dev),
            "total": torch.zeros(1, dtype=torch.int64, device=dev),
        }
    sp = stream_ptr(stream)
    s = stream if stream is not None else torch.cuda.current_stream()
    mv = np.ascontiguousarray(model_vec, dtype=np.float64)
    if events:
        events[0].record(s)
    N.check(L.bimine_mine_batch(dd.handle, N.ptr(mv, N._f64p), ctypes.byref(db.struct), ctypes.byref(db.plan), gap,
                                threshold, mismatch, bonus, sim.data_ptr(), db.t["out_off"].data_ptr(),
                                out["slots"].data_ptr(), out["counts"].data_ptr(), None, sp))
    if events:
        events[1].record(s)
    N.check(L.bimine_compact_matches(out["slots"].data_ptr(), db.t["out_off"].data_ptr(), out["counts"].data_ptr(),
                                     P, out["base"].data_ptr(), out["compact"].data_ptr(), out["total"].data_ptr(),
                                     sp))
    if events:
        events[2].record(s)
    return out


def nw_device(db: DeviceBatch, sim, gap: float, threshold: float, mismatch: float, bonus: float, out: dict,
              stream=None) -> None:
    """Standalone NW + traceback + filter over every pair of a scored batch
    (bimine_nw_mine_batch), for NW-only measurements."""
    torch = _torch()
    L = N.load()
    if "par" not in out:
        out["par"] = torch.tensor([gap, threshold], dtype=torch.float64, device=f"cuda:{db.device}")
    par = out["par"]
    N.check(L.bimine_nw_mine_batch(sim.data_ptr(), db.t["pair_sim_off"].data_ptr(), db.t["pair_n"].data_ptr(),
                                   db.t["pair_m"].data_ptr(), db.batch.n_pairs, db.max_n, db.max_m, 1,
                                   par.data_ptr(), par.data_ptr() + 8, mismatch, bonus, db.t["out_off"].data_ptr(),
                                   out["slots"].data_ptr(), out["counts"].data_ptr(), None, stream_ptr(stream)))


# ---------------------------------------------------------------------------
# host-buffer entry points
# ---------------------------------------------------------------------------

def _pinned_empty(n: int, dtype) -> np.ndarray:
    """Page-locked host array (torch's caching host allocator owns it)."""
    torch = _torch()
    dt = np.dtype(dtype)
    return torch.empty(n * dt.itemsize, dtype=torch.uint8, pin_memory=True).numpy().view(dt)


def mine_host(dd: DeviceDictionary, model_vec: np.ndarray, batch: PackedBatch, gap: float, threshold: float,
              mismatch: float, bonus: float, want_sim: bool = False, stream=None, out=None):
    """bimine_mine_host: H2D, score, NW, filter, compact, D2H.  Returns
    (counts[P], matches structured array, sim or None).

    `out`: optional dict reused across calls (a streaming caller's output
    buffers, in page-locked memory: the copy-out runs at full link speed and
    does not first-touch fresh pages); the returned arrays are views into it,
    valid until the next call with the same `out`."""
    L = N.load()
    torch = _torch()
    P = batch.n_pairs
    cap = int(np.minimum(batch.pair_n, batch.pair_m).sum(dtype=np.int64))
    if out is not None and out.get("counts") is not None and out["counts"].size >= max(P, 1) \
            and out["matches"].size >= max(cap, 1):
        counts, matches, total = out["counts"], out["matches"], out["total"]
    elif out is not None:
        grow = max(P, 1), max(cap, 1)
        if out.get("counts") is not None:  # amortise regrowth
            grow = max(grow[0], out["counts"].size * 5 // 4), max(grow[1], out["matches"].size * 5 // 4)
        out["counts"] = counts = _pinned_empty(grow[0], np.int32)
        out["matches"] = matches = _pinned_empty(grow[1], N.MATCH_DTYPE)
        out["total"] = total = _pinned_empty(1, np.int64)
    else:
        counts = np.empty(max(P, 1), dtype=np.int32)  # filled for every pair
        matches = np.empty(max(cap, 1), dtype=N.MATCH_DTYPE)  # the first `total` are filled
        total = np.zeros(1, dtype=np.int64)
    sim = np.empty(max(batch.n_cells, 1), dtype=np.float64) if want_sim else None
    cb = N.batch_struct_host(batch)
    mv = np.ascontiguousarray(model_vec, dtype=np.float64)
    with torch.cuda.device(dd.device):
        N.check(L.bimine_mine_host(dd.handle, N.ptr(mv, N._f64p), ctypes.byref(cb), gap, threshold, mismatch, bonus,
                                   N.ptr(counts, N._i32p), matches.ctypes.data, max(cap, 1), N.ptr(total, N._i64p),
                                   sim.ctypes.data if sim is not None else None, stream_ptr(stream)))
    return counts[:P], matches[: int(total[0])], (sim[: batch.n_cells] if sim is not None else None)


def score_host(dd: DeviceDictionary, model_vec: np.ndarray, batch: PackedBatch) -> np.ndarray:
    """Score matrices of a host batch (flat, at pair_sim_off)."""
    torch = _torch()
    with torch.cuda.device(dd.device):
        db = DeviceBatch(batch, dd.device)
        sim = torch.empty(max(batch.n_cells, 1), dtype=torch.float64, device=f"cuda:{dd.device}")
        score_device(dd, model_vec, db, sim)
        return sim[: batch.n_cells].cpu().numpy()


def features_host(dd: DeviceDictionary, model_vec: np.ndarray, batch: PackedBatch) -> np.ndarray:
    """The six features of every cell of a host batch (bimine_features_batch),
    [cells, 6] in pair_sim_off order."""
    torch = _torch()
    L = N.load()
    mv = np.ascontiguousarray(model_vec, dtype=np.float64)
    with torch.cuda.device(dd.device):
        db = DeviceBatch(batch, dd.device)
        dev = f"cuda:{dd.device}"
        sim = torch.empty(max(batch.n_cells, 1), dtype=torch.float64, device=dev)
        feats = torch.empty(max(batch.n_cells, 1) * 6, dtype=torch.float64, device=dev)
        N.check(L.bimine_features_batch(dd.handle, N.ptr(mv, N._f64p), ctypes.byref(db.struct), ctypes.byref(db.plan),
                                        sim.data_ptr(), feats.data_ptr(), stream_ptr(None)))
        return feats[: 6 * batch.n_cells].cpu().numpy().reshape(-1, 6)


def nw_steps_host(sims: list[np.ndarray], gaps: list[float], mismatch: float, bonus: float, device: int | None = None):
    """Full step lists for a list of matrices: [(codes uint8[k], score)]."""
    torch = _torch()
    L = N.load()
    if device is None:
        device = current_device()
    dev = f"cuda:{device}"
    n = np.array([s.shape[0] for s in sims], dtype=np.int32)
    m = np.array([s.shape[1] for s in sims], dtype=np.int32)
    cells = n.astype(np.int64) * m
    sim_off = np.zeros(len(sims), dtype=np.int64)
    np.cumsum(cells[:-1], out=sim_off[1:])
    step_off = np.zeros(len(sims), dtype=np.int64)
    np.cumsum((n + m)[:-1].astype(np.int64), out=step_off[1:])
    flat = np.concatenate([np.ascontiguousarray(s, dtype=np.float64).ravel() for s in sims])
    with torch.cuda.device(device):
        t_sim = torch.from_numpy(flat).to(dev)
        t_off = torch.from_numpy(sim_off).to(dev)
        t_n = torch.from_numpy(n).to(dev)
        t_m = torch.from_numpy(m).to(dev)
        t_gap = torch.tensor(np.asarray(gaps, dtype=np.float64)).to(dev)
        t_soff = torch.from_numpy(step_off).to(dev)
        t_steps = torch.empty(int((n + m).sum()), dtype=torch.uint8, device=dev)
        t_nsteps = torch.empty(len(sims), dtype=torch.int32, device=dev)
        t_score = torch.empty(len(sims), dtype=torch.float64, device=dev)
        N.check(L.bimine_nw_steps_batch(t_sim.data_ptr(), t_off.data_ptr(), t_n.data_ptr(), t_m.data_ptr(),
                                        len(sims), int(n.max()), int(m.max()), t_gap.data_ptr(), mismatch, bonus,
                                        t_soff.data_ptr(), t_steps.data_ptr(), t_nsteps.data_ptr(),
                                        t_score.data_ptr(), stream_ptr()))
        steps = t_steps.cpu().numpy()
        nsteps = t_nsteps.cpu().numpy()
        scores = t_score.cpu().numpy()
    return [(steps[step_off[k] : step_off[k] + nsteps[k]], float(scores[k])) for k in range(len(sims))]


def nw_fill_host(dp: np.ndarray, sim: np.ndarray, mismatch: float, bonus: float, gap: float) -> None:
    """The reference FFI contract (_nwcore.nw_fill): dp initialised by the caller."""
    L = N.load()
    if dp.dtype != np.float64 or not dp.flags.c_contiguous or not dp.flags.writeable:
        raise ValueError("dp must be a writable C-contiguous float64 array")
    sim = np.ascontiguousarray(sim, dtype=np.float64)
    n, m = sim.shape
    if dp.shape != (n + 1, m + 1):
        raise ValueError("dp must have shape (n + 1, m + 1)")
    N.check(L.bimine_nw_fill(N.ptr(dp, N._f64p), N.ptr(sim, N._f64p), n, m, mismatch, bonus, gap, None))


def exp_device(x: np.ndarray) -> np.ndarray:
    L = N.load()
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty_like(x)
    N.check(L.bimine_exp_device(N.ptr(x, N._f64p), N.ptr(y, N._f64p), x.size))
    return y


class DeviceTuner:
    """The tuning sweep's device state, kept across calls: the device batch
    and its plan, the score buffer, the per-(pair, trial) match slots, the
    trial parameters, the reference lists and page-locked staging for the
    inputs and the two result arrays.  A call uploads the batch from the
    staging (non-blocking copies on the tuner's stream), scores every pair
    once, aligns it under every trial in one launch (problem = pair * S +
    trial), runs the agreement NW on device and reads the results back with
    one synchronisation."""

    def __init__(self, dd: DeviceDictionary, model_vec: np.ndarray, batch: PackedBatch, thresholds, gaps,
                 mismatch: float, bonus: float, refs: list, stream=None):
        torch = _torch()
        self.torch = torch
        self.dd = dd
        self.device = dd.device
        self.batch = batch
        self.model = np.ascontiguousarray(model_vec, dtype=np.float64)
        self.mismatch, self.bonus = float(mismatch), float(bonus)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        dev = f"cuda:{self.device}"
        P, S = batch.n_pairs, len(gaps)
        self.P, self.S = P, S
        with torch.cuda.device(self.device):
            # page-locked staging of every input array; the device copies
            self.host = {f: torch.empty(max(getattr(batch, f).shape[0], 1), dtype=_torch_dtype(getattr(batch, f)),
                                        pin_memory=True) for f in _FIELDS}
            self.db = DeviceBatch(batch, self.device)
            self.sim = torch.empty(max(batch.n_cells, 1), dtype=torch.float64, device=dev)
            cap = np.minimum(batch.pair_n, batch.pair_m).astype(np.int64)
            self.cap_max = int(cap.max(initial=1))
            per_problem = np.repeat(cap, S)
            out_off = np.zeros(P * S, dtype=np.int64)
            if P * S > 1:
                np.cumsum(per_problem[:-1], out=out_off[1:])
            self.t_off = torch.from_numpy(out_off).to(dev)
            self.trials = (np.asarray(thresholds, dtype=np.float64).copy(), np.asarray(gaps, dtype=np.float64).copy())
            self.t_gap = torch.from_numpy(self.trials[1]).to(dev)
            self.t_thr = torch.from_numpy(self.trials[0]).to(dev)
            self.slots = torch.empty(max(int(per_problem.sum()), 1) * 16, dtype=torch.uint8, device=dev)
            self.counts = torch.empty(max(P * S, 1), dtype=torch.int32, device=dev)
            self.matched = torch.empty(max(P * S, 1), dtype=torch.int32, device=dev)
            self.h_counts = torch.empty(max(P * S, 1), dtype=torch.int32, pin_memory=True)
            self.h_matched = torch.empty(max(P * S, 1), dtype=torch.int32, pin_memory=True)
            self._refs = None
            self.set_refs(refs)

    def fits(self, batch: PackedBatch, n_settings: int) -> bool:
        """Same shapes as the tuner's batch (its plan and slot offsets hold)."""
        b = self.batch
        return (batch is b) or (
            n_settings == self.S and batch.n_pairs == b.n_pairs and batch.n_sentences == b.n_sentences
            and batch.n_tokens == b.n_tokens and np.array_equal(batch.pair_n, b.pair_n)
            and np.array_equal(batch.pair_m, b.pair_m) and np.array_equal(batch.sent_len, b.sent_len)
            and np.array_equal(batch.pair_sim_off, b.pair_sim_off))

    def set_refs(self, refs: list) -> None:
        if refs is self._refs:
            return
        self._refs = refs
        torch = self.torch
        dev = f"cuda:{self.device}"
        P = self.P
        ref_len = np.array([len(r) for r in refs], dtype=np.int32)
        ref_off = np.zeros(P, dtype=np.int64)
        if P > 1:
            np.cumsum(ref_len[:-1].astype(np.int64), out=ref_off[1:])
        ref_ij = np.fromiter(itertools.chain.from_iterable(itertools.chain.from_iterable(refs)), dtype=np.int32,
                             count=2 * int(ref_len.sum()))
        self.ref_max = int(ref_len.max(initial=1))
        self.t_rij = torch.from_numpy(ref_ij if ref_ij.size else np.zeros(2, np.int32)).to(dev)
        self.t_roff = torch.from_numpy(ref_off).to(dev)
        self.t_rlen = torch.from_numpy(ref_len).to(dev)

    def set_trials(self, thresholds, gaps) -> None:
        thr = np.asarray(thresholds, dtype=np.float64)
        gp = np.asarray(gaps, dtype=np.float64)
        if np.array_equal(thr, self.trials[0]) and np.array_equal(gp, self.trials[1]):
            return
        self.trials = (thr.copy(), gp.copy())
        with self.torch.cuda.stream(self.stream):
            self.t_thr.copy_(self.torch.from_numpy(self.trials[0]))
            self.t_gap.copy_(self.torch.from_numpy(self.trials[1]))

    def upload(self, batch: PackedBatch) -> None:
        """The batch's arrays into the staging (the library's threaded
        streaming copy), then non-blocking H2D copies on the tuner's stream
        (same shapes as the tuner's batch)."""
        torch = self.torch
        L = N.load()
        with torch.cuda.stream(self.stream):
            for f in _FIELDS:
                a = np.ascontiguousarray(getattr(batch, f))
                h = self.host[f]
                if a.shape[0]:
                    hv = h[: a.shape[0]].numpy()
                    if a.dtype != hv.dtype:
                        a = a.astype(hv.dtype)
                    N.check(L.bimine_host_copy(hv.ctypes.data, a.ctypes.data, a.nbytes))
                    self.db.t[f][: a.shape[0]].copy_(h[: a.shape[0]], non_blocking=True)

    def run_device(self, events=None) -> None:
        """Enqueue score -> NW (all trials) -> agreement on the stream."""
        L = N.load()
        sp = stream_ptr(self.stream)
        db = self.db
        if events:
            events[0].record(self.stream)
        score_device(self.dd, self.model, db, self.sim, self.stream)
        if events:
            events[1].record(self.stream)
        N.check(L.bimine_nw_mine_batch(self.sim.data_ptr(), db.t["pair_sim_off"].data_ptr(),
                                       db.t["pair_n"].data_ptr(), db.t["pair_m"].data_ptr(), self.P, db.max_n,
                                       db.max_m, self.S, self.t_gap.data_ptr(), self.t_thr.data_ptr(), self.mismatch,
                                       self.bonus, self.t_off.data_ptr(), self.slots.data_ptr(),
                                       self.counts.data_ptr(), None, sp))
        if events:
            events[2].record(self.stream)
        N.check(L.bimine_agreement_batch(self.slots.data_ptr(), self.t_off.data_ptr(), self.counts.data_ptr(),
                                         self.P, self.S, self.t_rij.data_ptr(), self.t_roff.data_ptr(),
                                         self.t_rlen.data_ptr(), self.cap_max, self.ref_max,
                                         self.matched.data_ptr(), sp))
        if events:
            events[3].record(self.stream)

    def results(self):
        """D2H of counts and agreements (one synchronisation)."""
        n = self.P * self.S
        with self.torch.cuda.stream(self.stream):
            self.h_counts[:n].copy_(self.counts[:n], non_blocking=True)
            self.h_matched[:n].copy_(self.matched[:n], non_blocking=True)
        self.stream.synchronize()
        return self.h_counts[:n].numpy().copy(), self.h_matched[:n].numpy().copy()


def _torch_dtype(a: np.ndarray):
    torch = _torch()
    return {np.dtype(np.int32): torch.int32, np.dtype(np.int64): torch.int64, np.dtype(np.uint8): torch.uint8}[a.dtype]


def tune_device(dd: DeviceDictionary, model_vec: np.ndarray, batch: PackedBatch, thresholds, gaps,
                mismatch: float, bonus: float, refs: list, stream=None, tuner: DeviceTuner | None = None):
    """Score every pair once, align it under every (threshold, gap) trial in
    one batched launch (problem = pair * S + trial) and compute each trial's
    agreement NW on device.  Returns (counts[P*S], matched[P*S]) on host.

    `tuner`: a DeviceTuner built for this batch's shapes (a caller sweeping
    repeatedly keeps one); its device buffers and plan are reused and the
    inputs are uploaded again from its page-locked staging."""
    if tuner is None or tuner.dd is not dd or not tuner.fits(batch, len(gaps)):
        tuner = DeviceTuner(dd, model_vec, batch, thresholds, gaps, mismatch, bonus, refs, stream=stream)
    else:
        tuner.upload(batch)
        tuner.set_refs(refs)
        tuner.set_trials(thresholds, gaps)
    tuner.run_device()
    return tuner.results()
