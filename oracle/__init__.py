"""float64 CPU oracle for the STCA forward under RLB (arXiv 2511.06077, §3.1-3.2).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product package ``paper_2511_06077_b200`` never imports it and
shares no code with it (the only shared module is ``workload``, the seeded
input generator, which holds none of the method's arithmetic).

The arithmetic lives in ``stca_oracle.c`` (plain C, f64, scalar loops,
``-O2 -ffp-contract=off``); this file is ctypes marshalling only.  See the C
file's header for the equation-by-equation citations.

Pinned by ``tests/test_oracle_pins.py`` (closed forms, special cases,
invariants, brute force, a library routine); DESIGN.md lists every pin.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Dict, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "stca_oracle.c")
_LIB = os.path.join(_HERE, "libstca_oracle.so")

OK, ERR_INVALID_ARG, ERR_SHAPE, ERR_OFFSETS, ERR_EMPTY_HISTORY, ERR_OOM = 0, -1, -2, -3, -4, -7


def build(force: bool = False) -> str:
    """Compile the oracle (gcc, -O2 -ffp-contract=off).  Building is not using it."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11",
                               "-fPIC", "-shared", "-pthread", "-o", _LIB, _SRC, "-lm"])
    return _LIB


class _Cfg(ctypes.Structure):
    _fields_ = [("d", ctypes.c_int32), ("h", ctypes.c_int32), ("r", ctypes.c_int32),
                ("M", ctypes.c_int32), ("L_infer", ctypes.c_int32), ("ln_eps", ctypes.c_double),
                ("with_z", ctypes.c_int32)]


_P = ctypes.POINTER(ctypes.c_double)


class _Layer(ctypes.Structure):
    _fields_ = [(n, _P) for n in ("hWu", "hWv", "hWo", "hg", "hb", "qWu", "qWv", "qWo", "qg", "qb",
                                  "WQ", "WK", "WV", "WO", "WC")]


class _Head(ctypes.Structure):
    _fields_ = [(n, _P) for n in ("WZ", "Wu", "Wv", "Wo")]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        i64p = ctypes.POINTER(ctypes.c_int64)
        _lib.oracle_forward.argtypes = [ctypes.POINTER(_Cfg), ctypes.POINTER(_Layer), ctypes.POINTER(_Head),
                                        _P, ctypes.c_int64, i64p, ctypes.c_int64, _P, ctypes.c_int64, i64p,
                                        _P, _P, ctypes.c_int, ctypes.c_int32, i64p]
        _lib.oracle_forward.restype = ctypes.c_int
        _lib.oracle_attention.argtypes = [_P, _P, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                          _P, _P, _P, _P, ctypes.c_int, _P]
        _lib.oracle_attention.restype = ctypes.c_int
        _lib.oracle_swigluffn.argtypes = [_P, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, _P, _P, _P, _P]
        _lib.oracle_layernorm.argtypes = [_P, ctypes.c_int64, ctypes.c_int32, _P, _P, ctypes.c_double, _P]
        _lib.oracle_softmax.argtypes = [_P, ctypes.c_int64, _P]
        _lib.oracle_suffix.argtypes = [i64p, ctypes.c_int64, ctypes.c_int32, i64p]
        _lib.oracle_validate.argtypes = [ctypes.POINTER(_Cfg), i64p, i64p, ctypes.c_int64, ctypes.c_int64,
                                         ctypes.c_int64, i64p]
        _lib.oracle_validate.restype = ctypes.c_int
    return _lib


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a: Optional[np.ndarray]):
    if a is None:
        return ctypes.cast(None, _P)
    return a.ctypes.data_as(_P)


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


# ---------------------------------------------------------------------------
# primitives (for the pins)
# ---------------------------------------------------------------------------

def swigluffn(x, Wu, Wv, Wo) -> np.ndarray:
    """Eq.(1), row-wise."""
    x = _f64(np.atleast_2d(x))
    Wu, Wv, Wo = _f64(Wu), _f64(Wv), _f64(Wo)
    n, d = x.shape
    rd = Wu.shape[1]
    out = np.empty((n, d), dtype=np.float64)
    lib().oracle_swigluffn(_ptr(x), n, d, rd, _ptr(Wu), _ptr(Wv), _ptr(Wo), _ptr(out))
    return out


def layernorm(x, g=None, b=None, eps: float = 1e-5) -> np.ndarray:
    x = _f64(np.atleast_2d(x))
    n, d = x.shape
    g = _f64(np.ones(d) if g is None else g)
    b = _f64(np.zeros(d) if b is None else b)
    out = np.empty_like(x)
    lib().oracle_layernorm(_ptr(x), n, d, _ptr(g), _ptr(b), eps, _ptr(out))
    return out


def softmax(s) -> np.ndarray:
    s = _f64(s)
    out = np.empty_like(s)
    lib().oracle_softmax(_ptr(s), s.shape[0], _ptr(out))
    return out


def attention(q, Xt, h: int, WQ, WK, WV, WO, form: int = 0) -> np.ndarray:
    """One query, one layer: Eq.(4)-(6) (form 0) or Eq.(13) (form 1)."""
    q, Xt = _f64(q), _f64(np.atleast_2d(Xt))
    WQ, WK, WV, WO = _f64(WQ), _f64(WK), _f64(WV), _f64(WO)
    L, d = Xt.shape
    o = np.empty(d, dtype=np.float64)
    rc = lib().oracle_attention(_ptr(q), _ptr(Xt), L, d, h, _ptr(WQ), _ptr(WK), _ptr(WV), _ptr(WO), form, _ptr(o))
    if rc != OK:
        raise OracleError(rc, -1)
    return o


def suffix_starts(hist_off, L_infer: int) -> np.ndarray:
    hist_off = _i64(hist_off)
    B = hist_off.shape[0] - 1
    out = np.empty(max(B, 0), dtype=np.int64)
    lib().oracle_suffix(hist_off.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), B, L_infer,
                        out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)))
    return out


class OracleError(RuntimeError):
    def __init__(self, status: int, index: int):
        super().__init__(f"oracle status {status} (request {index})")
        self.status, self.index = status, index


# ---------------------------------------------------------------------------
# full forward
# ---------------------------------------------------------------------------

def forward(weights: Dict[str, np.ndarray], *, d: int, h: int, r: int, M: int, X, hist_off, xt, tgt_off,
            L_infer: int = 0, ln_eps: float = 1e-5, with_z: bool = True, form: int = 0,
            nthreads: int = 1):
    """Z [Nt, M, d] and z [Nt, d] (or None) in float64.

    ``weights`` maps every role name of ``workload.weight_names`` (query roles
    included; use ``workload.full_weights`` for the shared reading) to an array.
    """
    keep = []

    def W(name, required=True):
        if name not in weights:
            if required:
                raise KeyError(name)
            return ctypes.cast(None, _P)
        a = _f64(weights[name]).reshape(-1)
        keep.append(a)
        return _ptr(a)

    layers = (_Layer * M)()
    for i in range(1, M + 1):
        Ly = layers[i - 1]
        p = f"L{i}."
        Ly.hWu, Ly.hWv, Ly.hWo = W(p + "hist.Wu"), W(p + "hist.Wv"), W(p + "hist.Wo")
        Ly.hg, Ly.hb = W(p + "hist.ln_g"), W(p + "hist.ln_b")
        Ly.qWu, Ly.qWv, Ly.qWo = W(p + "qry.Wu"), W(p + "qry.Wv"), W(p + "qry.Wo")
        Ly.qg = W("L1.qry.ln_g") if i == 1 else ctypes.cast(None, _P)
        Ly.qb = W("L1.qry.ln_b") if i == 1 else ctypes.cast(None, _P)
        Ly.WQ, Ly.WK, Ly.WV, Ly.WO = W(p + "WQ"), W(p + "WK"), W(p + "WV"), W(p + "WO")
        Ly.WC = W(p + "WC") if i >= 2 else ctypes.cast(None, _P)
    head = _Head()
    if with_z:
        head.WZ, head.Wu, head.Wv, head.Wo = W("z.WZ"), W("z.Wu"), W("z.Wv"), W("z.Wo")
    X, xt = _f64(X).reshape(-1, d), _f64(xt).reshape(-1, d)
    hist_off, tgt_off = _i64(hist_off), _i64(tgt_off)
    B = hist_off.shape[0] - 1
    T, Nt = X.shape[0], xt.shape[0]
    Z = np.zeros((Nt, M, d), dtype=np.float64)
    z = np.zeros((Nt, d), dtype=np.float64) if with_z else None
    cfg = _Cfg(d, h, r, M, L_infer, ln_eps, 1 if with_z else 0)
    bad = ctypes.c_int64(-1)
    i64p = ctypes.POINTER(ctypes.c_int64)
    rc = lib().oracle_forward(ctypes.byref(cfg), layers, ctypes.byref(head), _ptr(X), T,
                              hist_off.ctypes.data_as(i64p), B, _ptr(xt), Nt, tgt_off.ctypes.data_as(i64p),
                              _ptr(Z), _ptr(z), form, nthreads, ctypes.byref(bad))
    if rc != OK:
        raise OracleError(rc, bad.value)
    return Z, z


def forward_workload(wl, *, form: int = 0, nthreads: int = 1, requests=None, L_infer=None):
    """Run the oracle on a ``workload.Workload`` (optionally a subset of requests).

    Returns (Z, z, target_rows) where target_rows indexes the workload's target rows.
    """
    import workload as _w  # the shared seeded-input module (no method arithmetic)
    cfg = wl.cfg
    Li = cfg.L_infer if L_infer is None else L_infer
    if requests is None:
        X, hist_off, xt, tgt_off = wl.X, wl.hist_off, wl.xt, wl.tgt_off
        rows = np.arange(wl.Nt)
    else:
        requests = np.asarray(requests, dtype=np.int64)
        xs, ts, rows = [], [], []
        ho, to = [0], [0]
        for b in requests:
            s, e = wl.hist_off[b], wl.hist_off[b + 1]
            ts0, ts1 = wl.tgt_off[b], wl.tgt_off[b + 1]
            xs.append(wl.X[s:e]); ts.append(wl.xt[ts0:ts1]); rows.append(np.arange(ts0, ts1))
            ho.append(ho[-1] + (e - s)); to.append(to[-1] + (ts1 - ts0))
        X, xt = np.concatenate(xs), np.concatenate(ts)
        hist_off, tgt_off = np.array(ho), np.array(to)
        rows = np.concatenate(rows)
    Z, z = forward(_w.full_weights(wl), d=cfg.d, h=cfg.h, r=cfg.r, M=cfg.M, X=X, hist_off=hist_off, xt=xt,
                   tgt_off=tgt_off, L_infer=Li, with_z=cfg.with_z, form=form, nthreads=nthreads)
    return Z, z, rows
