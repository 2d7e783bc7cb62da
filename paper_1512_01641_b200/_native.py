"""ctypes binding of libbimine_b200.so (include/bimine_b200.h).

The CUDA library is the only compute path: there is no CPU fallback.
Importing this module never touches the GPU; the first call loads the
library and raises ``NativeUnavailable`` if it is missing or no CUDA
device is present, instead of silently computing elsewhere.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# BIMINE_LIB: load another build of the library (A/B kernel experiments)
LIB_PATH = os.environ.get("BIMINE_LIB") or os.path.join(HERE, "libbimine_b200.so")

_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)
_f64p = ctypes.POINTER(ctypes.c_double)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_vp = ctypes.c_void_p

MATCH_DTYPE = np.dtype([("score", "<f8"), ("i", "<i4"), ("j", "<i4")])

BIMINE_E_ARG, BIMINE_E_CUDA, BIMINE_E_LIMIT, BIMINE_E_NOMEM = -1, -2, -3, -4


class NativeUnavailable(RuntimeError):
    """The CUDA library (or a CUDA device) is not available."""


class BimineError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(f"bimine_b200 error {code}: {message}")
        self.code = code


class CBatch(ctypes.Structure):
    _fields_ = [
        ("n_pairs", ctypes.c_int64),
        ("n_sentences", ctypes.c_int64),
        ("n_tokens", ctypes.c_int64),
        ("tokens", _vp),
        ("sent_tok_off", _vp),
        ("sent_len", _vp),
        ("sent_uniq", _vp),
        ("sent_chars", _vp),
        ("pair_src", _vp),
        ("pair_n", _vp),
        ("pair_tgt", _vp),
        ("pair_m", _vp),
        ("pair_sim_off", _vp),
        ("token_bytes", ctypes.c_int32),
        ("sent_bytes", ctypes.c_int32),
    ]


class CDictView(ctypes.Structure):
    _fields_ = [
        ("n_rows", ctypes.c_int64),
        ("n_entries", ctypes.c_int64),
        ("row_ptr", _vp),
        ("tgt", _vp),
        ("prob", _vp),
    ]


class CPlan(ctypes.Structure):
    _fields_ = [
        ("max_n", ctypes.c_int32),
        ("max_m", ctypes.c_int32),
        ("max_uniq", ctypes.c_int32),
        ("max_len", ctypes.c_int32),
        ("n_tiles", ctypes.c_int64),
        ("n_long", ctypes.c_int64),
        ("long_max_n", ctypes.c_int32),
        ("long_max_m", ctypes.c_int32),
        ("n_large", ctypes.c_int64),
        ("n_cells", ctypes.c_int64),
        ("work_len", ctypes.c_int64),
        ("work", _vp),
        ("work_host", _vp),
    ]


# name -> (restype, argtypes); the complete exported surface of the header
SIGNATURES = {
    "bimine_last_error": (ctypes.c_char_p, []),
    "bimine_version": (ctypes.c_char_p, []),
    "bimine_nw_fill": (ctypes.c_int, [_f64p, _f64p, ctypes.c_int64, ctypes.c_int64, ctypes.c_double,
                                      ctypes.c_double, ctypes.c_double, _vp]),
    "bimine_nw_fill_wavefront": (ctypes.c_int, [_f64p, _f64p, ctypes.c_int64, ctypes.c_int64, ctypes.c_double,
                                                ctypes.c_double, ctypes.c_double, ctypes.c_int, _vp]),
    "bimine_dict_create": (ctypes.c_int, [_i32p, _i32p, _f64p, ctypes.c_int64, ctypes.POINTER(_vp)]),
    "bimine_dict_destroy": (ctypes.c_int, [_vp]),
    "bimine_dict_view_get": (ctypes.c_int, [_vp, ctypes.POINTER(CDictView)]),
    "bimine_dict_entries": (ctypes.c_int64, [_vp]),
    "bimine_plan_batch": (ctypes.c_int, [ctypes.POINTER(CBatch), _i64p, ctypes.c_int64, ctypes.POINTER(CPlan)]),
    "bimine_score_batch": (ctypes.c_int, [_vp, _f64p, ctypes.POINTER(CBatch), ctypes.POINTER(CPlan), _vp, _vp]),
    "bimine_mine_batch": (ctypes.c_int, [_vp, _f64p, ctypes.POINTER(CBatch), ctypes.POINTER(CPlan), ctypes.c_double,
                                         ctypes.c_double, ctypes.c_double, ctypes.c_double, _vp, _vp, _vp, _vp, _vp,
                                         _vp]),
    "bimine_nw_mine_batch": (ctypes.c_int, [_vp, _vp, _vp, _vp, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                            ctypes.c_int32, _vp, _vp, ctypes.c_double, ctypes.c_double, _vp, _vp,
                                            _vp, _vp, _vp]),
    "bimine_nw_steps_batch": (ctypes.c_int, [_vp, _vp, _vp, _vp, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                             _vp, ctypes.c_double, ctypes.c_double, _vp, _vp, _vp, _vp, _vp]),
    "bimine_agreement_batch": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int64, ctypes.c_int32, _vp, _vp, _vp,
                                              ctypes.c_int32, ctypes.c_int32, _vp, _vp]),
    "bimine_compact_matches": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int64, _vp, _vp, _vp, _vp]),
    "bimine_mine_host": (ctypes.c_int, [_vp, _f64p, ctypes.POINTER(CBatch), ctypes.c_double, ctypes.c_double,
                                        ctypes.c_double, ctypes.c_double, _i32p, _vp, ctypes.c_int64, _i64p,
                                        _vp, _vp]),
    "bimine_exp_device": (ctypes.c_int, [_f64p, _f64p, ctypes.c_int64]),
    "bimine_features_batch": (ctypes.c_int, [_vp, _f64p, ctypes.POINTER(CBatch), ctypes.POINTER(CPlan), _vp, _vp,
                                             _vp]),
    # device pointers (torch tensors' data_ptr)
    "bimine_lexicon_em": (ctypes.c_int, [_vp, _vp, ctypes.c_int64, ctypes.c_int32, _vp, _vp, ctypes.c_int64, _vp,
                                         _vp, _vp, _vp, ctypes.c_int32, _vp]),
    "bimine_vocab_create": (ctypes.c_int, [ctypes.POINTER(_vp)]),
    "bimine_vocab_destroy": (ctypes.c_int, [_vp]),
    "bimine_vocab_size": (ctypes.c_int64, [_vp]),
    "bimine_vocab_add_batch": (ctypes.c_int, [_vp, ctypes.c_char_p, _i64p, ctypes.c_int64, _i32p]),
    "bimine_vocab_word": (ctypes.c_int, [_vp, ctypes.c_int32, ctypes.POINTER(ctypes.c_char_p), _i64p]),
    "bimine_tokenize_batch": (ctypes.c_int, [_vp, ctypes.c_char_p, _i64p, ctypes.c_int64, _i32p, ctypes.c_int64,
                                             _i64p, _i32p, _i32p, _i32p]),
    "bimine_host_copy": (ctypes.c_int, [_vp, _vp, ctypes.c_int64]),
    "bimine_tokenize_ptrs": (ctypes.c_int, [_vp, _vp, _i64p, ctypes.c_int64, _i64p, _i32p, ctypes.c_int64, _i64p,
                                            _i32p, _i32p, _i32p]),
}

_lib = None
_lock = threading.Lock()


def load(require_gpu: bool = True):
    """Load the library (once).  Raises NativeUnavailable loudly."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeUnavailable(
                    f"{LIB_PATH} is not built; run `python -m paper_1512_01641_b200.build` "
                    "(there is no CPU fallback for the B200 path)"
                )
            L = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    if require_gpu:
        import torch

        if not torch.cuda.is_available():
            raise NativeUnavailable("no CUDA device: the bimine B200 path needs a GPU (no CPU fallback)")
    return _lib


def check(rc: int) -> None:
    if rc != 0:
        msg = _lib.bimine_last_error().decode() if _lib is not None else "?"
        raise BimineError(rc, msg)


def ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def batch_struct_host(b) -> CBatch:
    return CBatch(
        b.n_pairs, b.n_sentences, b.n_tokens,
        b.tokens.ctypes.data, b.sent_tok_off.ctypes.data, b.sent_len.ctypes.data, b.sent_uniq.ctypes.data,
        b.sent_chars.ctypes.data, b.pair_src.ctypes.data, b.pair_n.ctypes.data, b.pair_tgt.ctypes.data,
        b.pair_m.ctypes.data, b.pair_sim_off.ctypes.data, getattr(b, "token_bytes", 4),
        getattr(b, "sent_bytes", 4),
    )


def batch_struct_device(t: dict, n_pairs: int, n_sentences: int, n_tokens: int, token_bytes: int = 4) -> CBatch:
    """From a dict of device torch tensors named like PackedBatch fields."""
    return CBatch(
        n_pairs, n_sentences, n_tokens,
        t["tokens"].data_ptr(), t["sent_tok_off"].data_ptr(), t["sent_len"].data_ptr(), t["sent_uniq"].data_ptr(),
        t["sent_chars"].data_ptr(), t["pair_src"].data_ptr(), t["pair_n"].data_ptr(), t["pair_tgt"].data_ptr(),
        t["pair_m"].data_ptr(), t["pair_sim_off"].data_ptr(), token_bytes, 4,
    )
