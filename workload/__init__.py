"""Seeded synthetic inputs for the STCA-under-RLB forward (arXiv 2511.06077).

This module is the ONE piece of code shared by the oracle side (``oracle/``,
``tests/``) and the GPU side (``bench.py``, the binding's users).  It holds none
of the method's arithmetic: it only draws random numbers, rounds them to the
storage precision and lays them out.  Nothing here computes SwiGLU, LayerNorm,
attention, fusion or any other step of PAPER.md §3.1.

Recipe:

* one ``numpy.random.Generator(PCG64(seed))`` per workload, consumed in a fixed
  order: weights (``weight_names`` order) -> B Beta draws for the lengths ->
  history embeddings X (row-major) -> target embeddings x_t (row-major);
* dense weights ~ U(-1/sqrt(fan_in), 1/sqrt(fan_in)), fan_in = rows of the
  ``[in x out]`` matrix; LayerNorm gamma = 1, beta = 0 unless ``ln_affine``;
* X, x_t ~ N(0, 1) (float32 ziggurat), i.e. unit-scale embeddings;
* lengths: the paper's stochastic-length sampler, §3.3.1 Eq.(16)-(17)
  (P:L249-276): s ~ Beta(alpha, beta), beta = alpha (L_max - L_avg) / (L_avg -
  L_min), L_raw = L_min + s (L_max - L_min), rounded to the nearest multiple of
  8 (ties up), clamped to [8, L_max];
* bf16 configs: every value is rounded float32 -> bfloat16 (round to nearest
  even) and kept both as bit patterns (uint16) and as the float32 values those
  bits encode, so the oracle (which widens to f64) and the GPU see identical
  numbers.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, List, Optional

import numpy as np

__all__ = [
    "Config", "CONFIGS", "Workload", "make_workload", "weight_names",
    "weight_shapes", "beta_for", "sample_lengths", "bf16_bits", "bf16_round",
    "bits_to_f32",
]


@dataclasses.dataclass(frozen=True)
class Config:
    """Workload shape, BASELINE.json ``configs``."""
    name: str
    B: int                 # requests
    m: int                 # targets per request (RLB micro-batch size)
    d: int
    h: int
    r: int
    M: int                 # stacked layers
    dtype: str             # "fp32" | "bf16"
    L_fixed: int = 0       # >0: every history has this length
    L_min: int = 64
    L_max: int = 0
    L_avg: int = 0
    alpha: float = 0.02    # Beta shape, the paper's best
    L_infer: int = 0       # serving cap; 0 = no cap
    shared_ffn: bool = True   # DESIGN.md reading R5
    with_z: bool = True


CONFIGS: Dict[str, Config] = {
    "tiny": Config("tiny", B=1, m=4, d=32, h=1, r=4, M=2, dtype="fp32", L_fixed=64),
    "train": Config("train", B=1024, m=16, d=128, h=4, r=4, M=4, dtype="bf16",
                    L_min=64, L_max=4096, L_avg=2048),
    "serve": Config("serve", B=256, m=64, d=128, h=4, r=4, M=4, dtype="bf16",
                    L_fixed=10000, L_infer=10000),
    "capacity": Config("capacity", B=512, m=32, d=512, h=8, r=4, M=8, dtype="bf16",
                       L_min=64, L_max=10000, L_avg=2000),
    "multi": Config("multi", B=8192, m=8, d=128, h=4, r=4, M=4, dtype="bf16",
                    L_min=64, L_max=10000, L_avg=2000, L_infer=10000),
    "split1": Config("split1", B=1, m=64, d=128, h=4, r=4, M=4, dtype="bf16",
                     L_fixed=10000, L_infer=10000),
}


# --------------------------------------------------------------------------
# bf16 rounding (storage precision only; not method arithmetic)
# --------------------------------------------------------------------------

def bf16_bits(a: np.ndarray) -> np.ndarray:
    """float32 -> bfloat16 bit patterns, round to nearest even (finite inputs)."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    rounded = (u + np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))) >> np.uint32(16)
    return rounded.astype(np.uint16)


def bits_to_f32(b: np.ndarray) -> np.ndarray:
    """bfloat16 bit patterns -> the float32 values they encode (exact)."""
    return (np.ascontiguousarray(b, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def bf16_round(a: np.ndarray) -> np.ndarray:
    return bits_to_f32(bf16_bits(a))


# --------------------------------------------------------------------------
# weights
# --------------------------------------------------------------------------

def weight_names(M: int, shared_ffn: bool = True, with_z: bool = True) -> List[str]:
    """Names in draw order (the C-ABI's names, include/stca.h)."""
    names: List[str] = []
    for i in range(1, M + 1):
        names += [f"L{i}.hist.Wu", f"L{i}.hist.Wv", f"L{i}.hist.Wo",
                  f"L{i}.hist.ln_g", f"L{i}.hist.ln_b"]
        if not shared_ffn:
            names += [f"L{i}.qry.Wu", f"L{i}.qry.Wv", f"L{i}.qry.Wo"]
            if i == 1:
                names += ["L1.qry.ln_g", "L1.qry.ln_b"]
        names += [f"L{i}.WQ", f"L{i}.WK", f"L{i}.WV", f"L{i}.WO"]
        if i >= 2:
            names.append(f"L{i}.WC")
    if with_z:
        names += ["z.WZ", "z.Wu", "z.Wv", "z.Wo"]
    return names


def weight_shapes(d: int, r: int, M: int, shared_ffn: bool = True, with_z: bool = True):
    rd = r * d
    shapes = {}
    for n in weight_names(M, shared_ffn, with_z):
        leaf = n.split(".")[-1]
        if leaf in ("Wu", "Wv"):
            shapes[n] = (d, rd)
        elif leaf == "Wo":
            shapes[n] = (rd, d)
        elif leaf in ("ln_g", "ln_b"):
            shapes[n] = (1, d)
        elif leaf in ("WQ", "WK", "WV", "WO"):
            shapes[n] = (d, d)
        elif leaf == "WC":
            i = int(n.split(".")[0][1:])
            shapes[n] = (i * d, d)
        elif leaf == "WZ":
            shapes[n] = ((M + 1) * d, d)
        else:  # pragma: no cover
            raise KeyError(n)
    return shapes


# --------------------------------------------------------------------------
# lengths (§3.3.1, Eq. 16-17)
# --------------------------------------------------------------------------

def beta_for(alpha: float, L_min: int, L_max: int, L_avg: int) -> float:
    """Eq.(17): beta = alpha (L_max - L_avg) / (L_avg - L_min)."""
    return alpha * (L_max - L_avg) / (L_avg - L_min)


def round8(x: np.ndarray) -> np.ndarray:
    """Nearest multiple of 8, ties up."""
    return (np.floor(np.asarray(x, dtype=np.float64) / 8.0 + 0.5) * 8).astype(np.int64)


def sample_lengths(rng: np.random.Generator, cfg: Config, B: int) -> np.ndarray:
    if cfg.L_fixed:
        return np.full(B, cfg.L_fixed, dtype=np.int64)
    beta = beta_for(cfg.alpha, cfg.L_min, cfg.L_max, cfg.L_avg)
    s = rng.beta(cfg.alpha, beta, size=B)
    L_raw = cfg.L_min + s * (cfg.L_max - cfg.L_min)          # Eq.(16)
    return np.clip(round8(L_raw), 8, cfg.L_max).astype(np.int64)


# --------------------------------------------------------------------------
# the workload
# --------------------------------------------------------------------------

@dataclasses.dataclass
class Workload:
    cfg: Config
    seed: int
    weights: Dict[str, np.ndarray]        # float32 values (bf16-exact for bf16 configs)
    lengths: np.ndarray                   # int64 [B]
    hist_off: np.ndarray                  # int64 [B+1]
    tgt_off: np.ndarray                   # int64 [B+1]
    X: np.ndarray                         # float32 [T x d]
    xt: np.ndarray                        # float32 [N_t x d]
    X_bits: Optional[np.ndarray] = None   # uint16 [T x d] (bf16 configs)
    xt_bits: Optional[np.ndarray] = None  # uint16 [N_t x d]

    @property
    def T(self) -> int:
        return int(self.hist_off[-1])

    @property
    def Nt(self) -> int:
        return int(self.tgt_off[-1])


def _normal_rows(rng: np.random.Generator, rows: int, d: int, chunk_rows: int = 1 << 16) -> np.ndarray:
    out = np.empty((rows, d), dtype=np.float32)
    for s in range(0, rows, chunk_rows):
        e = min(rows, s + chunk_rows)
        out[s:e] = rng.standard_normal((e - s, d), dtype=np.float32)
    return out


def _normal_rows_bits(rng: np.random.Generator, rows: int, d: int, chunk_rows: int = 1 << 16) -> np.ndarray:
    """The same draws as _normal_rows, kept only as bf16 bit patterns (chunk by chunk: no float32 copy
    of the whole matrix is ever held)."""
    out = np.empty((rows, d), dtype=np.uint16)
    for s in range(0, rows, chunk_rows):
        e = min(rows, s + chunk_rows)
        out[s:e] = bf16_bits(rng.standard_normal((e - s, d), dtype=np.float32)).reshape(e - s, d)
    return out


def make_workload(cfg, seed: int = 0, B: Optional[int] = None, *, ln_affine: bool = False,
                  wq_scale: float = 1.0, lengths: Optional[np.ndarray] = None,
                  m: Optional[int] = None, bits_only: bool = False) -> Workload:
    """Draw one workload.  ``B``/``m``/``lengths`` override the config (tests).  ``bits_only`` (bf16
    configs): keep X only as bf16 bit patterns (``X`` is None; ``subset`` widens the rows it needs),
    for the multi-GB bench workloads.  The draws are identical either way."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    B = cfg.B if B is None else int(B)
    m = cfg.m if m is None else int(m)
    rng = np.random.Generator(np.random.PCG64(seed))
    bf16 = cfg.dtype == "bf16"
    rnd = bf16_round if bf16 else (lambda a: np.asarray(a, dtype=np.float32))

    weights: Dict[str, np.ndarray] = {}
    for name, (rows, cols) in weight_shapes(cfg.d, cfg.r, cfg.M, cfg.shared_ffn, cfg.with_z).items():
        leaf = name.split(".")[-1]
        if leaf == "ln_g":
            w = (1.0 + 0.1 * rng.standard_normal((rows, cols))) if ln_affine else np.ones((rows, cols))
        elif leaf == "ln_b":
            w = (0.1 * rng.standard_normal((rows, cols))) if ln_affine else np.zeros((rows, cols))
        else:
            a = 1.0 / math.sqrt(rows)
            w = rng.uniform(-a, a, size=(rows, cols))
            if leaf == "WQ":
                w = w * wq_scale
        weights[name] = rnd(w.astype(np.float32))

    if lengths is None:
        lengths = sample_lengths(rng, cfg, B)
    lengths = np.asarray(lengths, dtype=np.int64)
    assert lengths.shape == (B,)
    hist_off = np.zeros(B + 1, dtype=np.int64)
    np.cumsum(lengths, out=hist_off[1:])
    tgt_off = np.arange(B + 1, dtype=np.int64) * m
    T, Nt = int(hist_off[-1]), int(tgt_off[-1])

    if bf16 and bits_only:
        X_bits = _normal_rows_bits(rng, T, cfg.d)
        xt_bits = _normal_rows_bits(rng, Nt, cfg.d)
        return Workload(cfg=cfg, seed=seed, weights=weights, lengths=lengths, hist_off=hist_off,
                        tgt_off=tgt_off, X=None, xt=bits_to_f32(xt_bits).reshape(Nt, cfg.d), X_bits=X_bits,
                        xt_bits=xt_bits)
    X = _normal_rows(rng, T, cfg.d)
    xt = _normal_rows(rng, Nt, cfg.d)
    X_bits = xt_bits = None
    if bf16:
        X_bits, xt_bits = bf16_bits(X), bf16_bits(xt)
        X, xt = bits_to_f32(X_bits).reshape(T, cfg.d), bits_to_f32(xt_bits).reshape(Nt, cfg.d)
        X_bits, xt_bits = X_bits.reshape(T, cfg.d), xt_bits.reshape(Nt, cfg.d)
    return Workload(cfg=cfg, seed=seed, weights=weights, lengths=lengths, hist_off=hist_off,
                    tgt_off=tgt_off, X=X, xt=xt, X_bits=X_bits, xt_bits=xt_bits)


def weight_aliases(cfg: Config) -> Dict[str, str]:
    """Shared reading R5: the query-path FFN/LN of layer i is the history FFN/LN of layer i."""
    if not cfg.shared_ffn:
        return {}
    al = {}
    for i in range(1, cfg.M + 1):
        for leaf in ("Wu", "Wv", "Wo"):
            al[f"L{i}.qry.{leaf}"] = f"L{i}.hist.{leaf}"
    al["L1.qry.ln_g"] = "L1.hist.ln_g"
    al["L1.qry.ln_b"] = "L1.hist.ln_b"
    return al


def full_weights(wl: Workload) -> Dict[str, np.ndarray]:
    """All role names (query roles resolved through the shared-reading aliases)."""
    w = dict(wl.weights)
    for k, v in weight_aliases(wl.cfg).items():
        w[k] = wl.weights[v]
    return w


def subset(wl: Workload, requests, with_f32: bool = True) -> Workload:
    """The workload restricted to ``requests`` (in the given order): their history rows and target
    rows back to back, offsets rebuilt.  Pure row selection (a request shard of a data-parallel rank,
    or the oracle's sample); no arithmetic."""
    req = np.asarray(requests, dtype=np.int64)
    L = wl.lengths[req]
    m = np.diff(wl.tgt_off)[req]
    hist_off = np.zeros(len(req) + 1, dtype=np.int64)
    np.cumsum(L, out=hist_off[1:])
    tgt_off = np.zeros(len(req) + 1, dtype=np.int64)
    np.cumsum(m, out=tgt_off[1:])

    def rows(off, idx):
        if len(idx) == 0:
            return np.zeros(0, dtype=np.int64)
        return np.concatenate([np.arange(off[b], off[b + 1], dtype=np.int64) for b in idx])
    hr, tr = rows(wl.hist_off, req), rows(wl.tgt_off, req)
    d = wl.cfg.d
    X_bits = wl.X_bits[hr] if wl.X_bits is not None else None
    xt_bits = wl.xt_bits[tr] if wl.xt_bits is not None else None
    if X_bits is not None:
        X = bits_to_f32(X_bits).reshape(-1, d) if with_f32 else None
        xt = bits_to_f32(xt_bits).reshape(-1, d)
    else:
        X, xt = wl.X[hr], wl.xt[tr]
    return Workload(cfg=wl.cfg, seed=wl.seed, weights=wl.weights, lengths=L, hist_off=hist_off, tgt_off=tgt_off,
                    X=X, xt=xt, X_bits=X_bits, xt_bits=xt_bits)
