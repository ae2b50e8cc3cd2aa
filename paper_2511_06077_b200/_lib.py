"""ctypes declarations of include/stca.h (marshalling only)."""
from __future__ import annotations

import ctypes
import os

import numpy as np

# STCA_LIB: another in-tree build of the same library (A/B experiments only)
LIB_PATH = os.environ.get("STCA_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libstca.so")
STCA_BF16, STCA_FP32 = 0, 1

EXCHANGE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                               ctypes.c_void_p)
# stca_alloc_fn / stca_free_fn (working-buffer provider)
ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int32, ctypes.c_void_p)
FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p)
PHASES = ["project", "attention", "merge", "target", "forward"]  # STCA_PH_* order


class _Config(ctypes.Structure):
    _fields_ = [("d", ctypes.c_int32), ("h", ctypes.c_int32), ("r", ctypes.c_int32), ("M", ctypes.c_int32),
                ("L_infer", ctypes.c_int32), ("ln_eps", ctypes.c_float), ("dtype", ctypes.c_int32),
                ("with_z", ctypes.c_int32), ("device", ctypes.c_int32), ("chunk_keys", ctypes.c_int32),
                ("split_rank", ctypes.c_int32), ("split_world", ctypes.c_int32), ("exchange", EXCHANGE_FN),
                ("exchange_ctx", ctypes.c_void_p), ("dev_alloc", ALLOC_FN), ("dev_free", FREE_FN),
                ("alloc_ctx", ctypes.c_void_p)]


class _Tensor(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char_p), ("data", ctypes.POINTER(ctypes.c_float)), ("rows", ctypes.c_int64),
                ("cols", ctypes.c_int64)]


class _Grad(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char_p), ("grad", ctypes.c_void_p)]


class _EmbedTables(ctypes.Structure):
    _fields_ = [("video", ctypes.c_void_p), ("n_video", ctypes.c_int64), ("action", ctypes.c_void_p),
                ("n_action", ctypes.c_int64), ("position", ctypes.c_void_p), ("n_position", ctypes.c_int64),
                ("tdelta", ctypes.c_void_p), ("n_tdelta", ctypes.c_int64)]


class StcaError(RuntimeError):
    def __init__(self, status: int, message: str = ""):
        super().__init__(f"{status_string(status)} ({status}): {message}")
        self.status, self.message = status, message


_lib = None
_I64P = ctypes.POINTER(ctypes.c_int64)

SYMBOLS = ["stca_create", "stca_project_history", "stca_forward", "stca_destroy", "stca_last_error",
           "stca_status_string", "stca_abi_version", "stca_validate_offsets", "stca_plan_suffix",
           "stca_plan_chunks", "stca_plan_attention", "stca_plan_shards", "stca_kernel_launches",
           "stca_plan_split", "stca_plan_persistent", "stca_read_cache", "stca_rlb_allocate", "stca_rlb_compact",
           "stca_profile", "stca_profile_read", "stca_session_open", "stca_project_history_session",
           "stca_encode_history", "stca_attention_backward", "stca_history_backward", "stca_backward",
           "stca_split_peer_export", "stca_split_peer_attach", "stca_ipc_open", "stca_ipc_close",
           "stca_set_attention_form"]


def lib():
    """Load libstca.so (fails loudly if it was not built: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2511_06077_b200.build` "
                              "(or __graft_entry__.build()); there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        L.stca_create.argtypes = [ctypes.POINTER(_Config), ctypes.POINTER(_Tensor), ctypes.c_int32,
                                  ctypes.POINTER(ctypes.c_void_p)]
        L.stca_create.restype = ctypes.c_int32
        L.stca_project_history.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, _I64P, ctypes.c_int64,
                                           ctypes.c_void_p]
        L.stca_project_history.restype = ctypes.c_int32
        L.stca_forward.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, _I64P, ctypes.c_int64,
                                   ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.stca_forward.restype = ctypes.c_int32
        L.stca_destroy.argtypes = [ctypes.c_void_p]
        L.stca_destroy.restype = None
        L.stca_last_error.argtypes = [ctypes.c_void_p]
        L.stca_last_error.restype = ctypes.c_char_p
        L.stca_status_string.argtypes = [ctypes.c_int32]
        L.stca_status_string.restype = ctypes.c_char_p
        L.stca_abi_version.restype = ctypes.c_int32
        L.stca_kernel_launches.restype = ctypes.c_int64
        L.stca_validate_offsets.argtypes = [_I64P, _I64P, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _I64P]
        L.stca_validate_offsets.restype = ctypes.c_int32
        L.stca_plan_suffix.argtypes = [_I64P, ctypes.c_int64, ctypes.c_int32, _I64P]
        L.stca_plan_suffix.restype = None
        L.stca_plan_chunks.argtypes = [ctypes.c_int64, ctypes.c_int32, _I64P]
        L.stca_plan_chunks.restype = ctypes.c_int32
        L.stca_plan_attention.argtypes = [_I64P, _I64P, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                          ctypes.c_int32, _I64P, ctypes.c_int64]
        L.stca_plan_attention.restype = ctypes.c_int64
        L.stca_plan_shards.argtypes = [_I64P, ctypes.c_int64, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32)]
        L.stca_plan_shards.restype = None
        L.stca_plan_split.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _I64P, _I64P]
        L.stca_plan_split.restype = None
        L.stca_plan_persistent.argtypes = [_I64P, ctypes.c_int64, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32),
                                           ctypes.POINTER(ctypes.c_int32)]
        L.stca_plan_persistent.restype = None
        L.stca_rlb_allocate.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                                        ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_void_p]
        L.stca_rlb_allocate.restype = ctypes.c_int32
        L.stca_rlb_compact.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.stca_rlb_compact.restype = ctypes.c_int32
        L.stca_read_cache.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                                      ctypes.c_void_p]
        L.stca_read_cache.restype = ctypes.c_int
        L.stca_debug_capture.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p]
        L.stca_debug_capture.restype = ctypes.c_int32
        L.stca_encode_history.argtypes = [ctypes.POINTER(_EmbedTables), ctypes.c_int32, ctypes.c_int32,
                                          ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                          ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                                          ctypes.c_void_p]
        L.stca_encode_history.restype = ctypes.c_int32
        L.stca_attention_backward.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, _I64P,
                                              ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.stca_attention_backward.restype = ctypes.c_int32
        L.stca_history_backward.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int64] + \
            [ctypes.c_void_p] * 8
        L.stca_history_backward.restype = ctypes.c_int32
        L.stca_backward.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, _I64P, ctypes.c_int64,
                                    ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                    ctypes.POINTER(_Grad), ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p,
                                    ctypes.c_void_p, ctypes.c_void_p]
        L.stca_backward.restype = ctypes.c_int32
        L.stca_split_peer_export.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.POINTER(ctypes.c_void_p),
                                             ctypes.c_void_p]
        L.stca_split_peer_export.restype = ctypes.c_int32
        L.stca_split_peer_attach.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]
        L.stca_split_peer_attach.restype = ctypes.c_int32
        L.stca_ipc_open.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.POINTER(ctypes.c_void_p)]
        L.stca_ipc_open.restype = ctypes.c_int32
        L.stca_ipc_close.argtypes = [ctypes.c_void_p]
        L.stca_ipc_close.restype = ctypes.c_int32
        L.stca_set_attention_form.argtypes = [ctypes.c_void_p, ctypes.c_int32]
        L.stca_set_attention_form.restype = ctypes.c_int32
        L.stca_session_open.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
        L.stca_session_open.restype = ctypes.c_int32
        L.stca_project_history_session.argtypes = [ctypes.c_void_p, _I64P, _I64P, ctypes.c_void_p, ctypes.c_int64,
                                                   _I64P, ctypes.c_int64, _I64P, ctypes.c_void_p]
        L.stca_project_history_session.restype = ctypes.c_int32
        L.stca_profile.argtypes = [ctypes.c_void_p, ctypes.c_int32]
        L.stca_profile.restype = ctypes.c_int32
        L.stca_profile_read.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), _I64P]
        L.stca_profile_read.restype = ctypes.c_int32
        if L.stca_abi_version() != 2:
            raise ImportError(f"{LIB_PATH}: ABI version {L.stca_abi_version()}, this binding speaks 2 (rebuild)")
        _lib = L
    return _lib


def status_string(s: int) -> str:
    try:
        return lib().stca_status_string(s).decode()
    except ImportError:  # pragma: no cover
        return str(s)


def _p64(a: np.ndarray):
    return a.ctypes.data_as(_I64P)


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64))


def validate_offsets(hist_off, tgt_off, T: int, Nt: int):
    h, t = _i64(hist_off), _i64(tgt_off)
    bad = ctypes.c_int64(-1)
    rc = lib().stca_validate_offsets(_p64(h), _p64(t), h.shape[0] - 1, T, Nt, ctypes.byref(bad))
    return rc, bad.value


def plan_suffix(hist_off, L_infer: int) -> np.ndarray:
    h = _i64(hist_off)
    out = np.zeros(max(h.shape[0] - 1, 0), dtype=np.int64)
    lib().stca_plan_suffix(_p64(h), h.shape[0] - 1, L_infer, _p64(out))
    return out


def plan_chunks(L: int, chunk_keys: int = 0):
    cl = ctypes.c_int64(0)
    n = lib().stca_plan_chunks(L, chunk_keys, ctypes.byref(cl))
    return n, cl.value


def plan_attention(hist_len, tgt_off, h: int, qtile: int, chunk_keys: int = 0) -> np.ndarray:
    hl, t = _i64(hist_len), _i64(tgt_off)
    B = hl.shape[0]
    n = lib().stca_plan_attention(_p64(hl), _p64(t), B, h, qtile, chunk_keys, None, 0)
    out = np.zeros((max(n, 1), 6), dtype=np.int64)
    lib().stca_plan_attention(_p64(hl), _p64(t), B, h, qtile, chunk_keys, _p64(out), n)
    return out[:n]


def plan_persistent(cost, n_ctas: int):
    """(cta_off [n_ctas + 1], cta_items [n], bin [n]) of the persistent attention schedule."""
    c = _i64(cost)
    n = c.shape[0]
    lst = np.zeros(n_ctas + 1 + n, dtype=np.int32)
    b = np.zeros(n, dtype=np.int32)
    i32p = ctypes.POINTER(ctypes.c_int32)
    lib().stca_plan_persistent(_p64(c), n, n_ctas, lst.ctypes.data_as(i32p), b.ctypes.data_as(i32p))
    return lst[:n_ctas + 1], lst[n_ctas + 1:], b


def plan_shards(cost, n_parts: int) -> np.ndarray:
    c = _i64(cost)
    out = np.zeros(c.shape[0], dtype=np.int32)
    lib().stca_plan_shards(_p64(c), c.shape[0], n_parts, out.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))
    return out


def kernel_launches() -> int:
    """Process-wide number of kernels libstca has launched (bench: gpu_launches)."""
    return int(lib().stca_kernel_launches())


def plan_split(L: int, chunk_keys: int, G: int, g: int):
    """(own0, olen): the key range rank g of G owns in split-history mode."""
    a, b = ctypes.c_int64(0), ctypes.c_int64(0)
    lib().stca_plan_split(L, chunk_keys, G, g, ctypes.byref(a), ctypes.byref(b))
    return a.value, b.value
