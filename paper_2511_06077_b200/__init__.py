"""B200-native STCA forward under Request-Level Batching (arXiv 2511.06077).

Thin ctypes binding over ``libstca.so`` (the C ABI declared in ``include/stca.h``).
This module only marshals arguments: every step of the path runs in the library's
CUDA kernels.  There is no CPU fallback; if the library is missing, importing
this package raises.

    import paper_2511_06077_b200 as stca
    m = stca.STCA(weights, d=128, h=4, r=4, M=4, L_infer=10000, dtype="bf16")
    m.project_history(X, hist_off)        # X: torch CUDA tensor (bf16/uint16 or fp32) or host numpy
    m.forward(xt, tgt_off, out_Z, out_z)  # outputs: float32 CUDA tensors or host numpy arrays
"""
from __future__ import annotations

import ctypes
import os
from typing import Dict, Optional

import numpy as np

from ._lib import (STCA_BF16, STCA_FP32, StcaError, lib, plan_attention, plan_chunks, plan_persistent, plan_shards,  # noqa: F401,E501
                   plan_split, plan_suffix, status_string, validate_offsets, kernel_launches, EXCHANGE_FN, ALLOC_FN,
                   FREE_FN, PHASES, _Config, _Tensor, _EmbedTables, _Grad, LIB_PATH)

__all__ = ["STCA", "StcaError", "plan_attention", "plan_chunks", "plan_persistent", "plan_shards", "plan_split", "plan_suffix",
           "validate_offsets", "status_string", "LIB_PATH", "nccl_exchange", "ThreadExchange", "rlb_allocate",
           "rlb_compact", "encode_history"]


def _ptr(x) -> int:
    """Address of a torch tensor (device or host) or a numpy array (host)."""
    if x is None:
        return 0
    if isinstance(x, np.ndarray):
        if not x.flags["C_CONTIGUOUS"]:
            raise ValueError("arrays must be C-contiguous")
        return x.ctypes.data
    if hasattr(x, "data_ptr"):
        if not x.is_contiguous():
            raise ValueError("tensors must be contiguous")
        return x.data_ptr()
    raise TypeError(f"unsupported buffer type {type(x)}")


def _stream(stream) -> int:
    if stream is not None:
        return int(stream) if isinstance(stream, int) else int(stream.cuda_stream)
    try:
        import torch
        if torch.cuda.is_available():
            return int(torch.cuda.current_stream().cuda_stream)
    except Exception:  # pragma: no cover
        pass
    return 0


def _is_cuda(x) -> bool:
    return bool(getattr(x, "is_cuda", False))


def _synchronize(stream) -> None:
    """Wait for `stream` (torch stream, raw cudaStream_t int, or None = torch's current stream)."""
    import torch
    if stream is None:
        torch.cuda.current_stream().synchronize()
    elif isinstance(stream, int):
        torch.cuda.ExternalStream(stream).synchronize()
    else:
        stream.synchronize()


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64))


def _torch_allocator():
    """stca_alloc_fn / stca_free_fn over PyTorch's CUDA caching allocator (stream-ordered blocks)."""
    import torch

    def alloc(ctx, nbytes, device, stream):
        try:
            return torch.cuda.caching_allocator_alloc(int(nbytes), device=int(device), stream=int(stream or 0))
        except Exception:  # OOM -> NULL -> STCA_ERR_OOM
            return None

    def free(ctx, ptr, device, stream):
        try:
            torch.cuda.caching_allocator_delete(int(ptr))
        except Exception:  # pragma: no cover  (interpreter shutdown)
            pass
    return ALLOC_FN(alloc), FREE_FN(free)


class STCA:
    """One handle = one device's copy of the weights + the projected history cache."""

    def __init__(self, weights: Dict[str, np.ndarray], *, d: int, h: int, r: int, M: int, L_infer: int = 0,
                 dtype: str = "bf16", with_z: bool = True, device: int = 0, chunk_keys: int = 0,
                 ln_eps: float = 1e-5, split_rank: int = 0, split_world: int = 1, exchange=None,
                 allocator: str = "torch"):
        """allocator: "torch" (working buffers from PyTorch's caching allocator) or "cuda" (the
        library's stream-ordered CUDA pool)."""
        self.d, self.h, self.r, self.M, self.with_z = d, h, r, M, with_z
        self._device = device
        self.dtype = dtype
        cfg = _Config()
        cfg.d, cfg.h, cfg.r, cfg.M = d, h, r, M
        cfg.L_infer = L_infer
        cfg.ln_eps = ln_eps
        cfg.dtype = STCA_BF16 if dtype == "bf16" else STCA_FP32
        cfg.with_z = 1 if with_z else 0
        cfg.device = device
        cfg.chunk_keys = chunk_keys
        cfg.split_rank, cfg.split_world = split_rank, split_world
        self._exchange_cb = None
        if exchange is not None:
            self._exchange_cb = EXCHANGE_FN(exchange)
            cfg.exchange = self._exchange_cb
        self._alloc_cbs = None
        if allocator == "torch":
            self._alloc_cbs = _torch_allocator()
            cfg.dev_alloc, cfg.dev_free = self._alloc_cbs
        elif allocator != "cuda":
            raise ValueError(f"allocator must be 'torch' or 'cuda', not {allocator!r}")
        # weights: host float32; identical array objects keep identical pointers (reading R5 aliasing)
        conv, keep = {}, []
        self._shapes = {}
        tens = (_Tensor * len(weights))()
        for i, (name, arr) in enumerate(weights.items()):
            key = id(arr)
            if key not in conv:
                a = np.ascontiguousarray(np.asarray(arr, dtype=np.float32))
                conv[key] = a
            a = conv[key]
            bname = name.encode()
            keep.append(bname)
            rows, cols = (1, a.size) if a.ndim == 1 else a.shape
            self._shapes[name] = (rows, cols)
            tens[i].name = bname
            tens[i].data = a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))
            tens[i].rows, tens[i].cols = rows, cols
        handle = ctypes.c_void_p()
        rc = lib().stca_create(ctypes.byref(cfg), tens, len(weights), ctypes.byref(handle))
        if rc != 0:
            raise StcaError(rc, lib().stca_last_error(None).decode())
        self._h = handle
        self._B = None

    # -- lifecycle --
    def close(self):
        """Destroys the handle.  Split-history over peer memory: every rank must be done with the buffers
        (a barrier) before any rank closes."""
        for p in getattr(self, "_ipc", []):
            lib().stca_ipc_close(ctypes.c_void_p(p))
        self._ipc = []
        if getattr(self, "_h", None):
            lib().stca_destroy(self._h)
            self._h = None

    def set_attention_form(self, form: str) -> None:
        """"reordered" (Eq.(13), default) or "standard" (Eq.(12): K/V per head materialised; NEXT-3 variant)."""
        self._check(lib().stca_set_attention_form(self._h, {"reordered": 0, "standard": 1}[form]))

    # ---- split-history over peer memory (stca_split_peer_*) ----
    def split_peer_export(self, capacity_bytes: int = 64 << 20):
        """Allocates this rank's exchange buffer; returns (device address, 64-byte IPC handle)."""
        base = ctypes.c_void_p()
        hd = (ctypes.c_uint8 * 64)()
        self._check(lib().stca_split_peer_export(self._h, int(capacity_bytes), ctypes.byref(base), hd))
        return int(base.value), bytes(hd)

    def split_peer_attach(self, bases) -> None:
        """bases: the G ranks' exchange buffers as device addresses valid in this process, rank order."""
        arr = (ctypes.c_void_p * len(bases))(*[ctypes.c_void_p(int(b)) for b in bases])
        self._check(lib().stca_split_peer_attach(self._h, arr))

    def split_peer_setup(self, capacity_bytes: int = 64 << 20, group=None) -> None:
        """One process per GPU (torch.distributed initialised, split_rank == the group rank): export, all-gather
        the IPC handles (setup only, never on the data path), map the peers' buffers, attach, barrier."""
        import torch.distributed as dist
        base, hd = self.split_peer_export(capacity_bytes)
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        handles = [None] * world
        dist.all_gather_object(handles, hd, group=group)
        bases, self._ipc = [], []
        for g, hg in enumerate(handles):
            if g == rank:
                bases.append(base)
                continue
            ptr = ctypes.c_void_p()
            buf = (ctypes.c_uint8 * 64).from_buffer_copy(hg)
            self._check(lib().stca_ipc_open(buf, int(self._device), ctypes.byref(ptr)))
            self._ipc.append(int(ptr.value))
            bases.append(int(ptr.value))
        self.split_peer_attach(bases)
        dist.barrier(group)

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        if rc != 0:
            raise StcaError(rc, lib().stca_last_error(self._h).decode())

    def debug_capture(self, layer: int, U, Y) -> None:
        """Test hook: the next forward copies layer `layer`'s U and Y (storage dtype, [Nt h x d]) into the
        given CUDA tensors."""
        self._check(lib().stca_debug_capture(self._h, int(layer), ctypes.c_void_p(_ptr(U)), ctypes.c_void_p(_ptr(Y))))

    # -- per-phase device timing (stca_profile) --
    PROF_EVENTS, PROF_TWICE_ATTENTION, PROF_TWICE_PROJECT, PROF_EVENTS_TARGET = 1, 2, 4, 8

    def profile(self, enable=True) -> None:
        """True / False: per-phase event regions; an int: the STCA_PROF_* bit mask (include/stca.h)."""
        mask = int(enable) if not isinstance(enable, bool) else (1 if enable else 0)
        self._check(lib().stca_profile(self._h, mask))

    def profile_read(self):
        """{phase: (total ms, regions)} since the last read (waits for the recorded events)."""
        ms = (ctypes.c_double * len(PHASES))()
        n = np.zeros(len(PHASES), dtype=np.int64)
        self._check(lib().stca_profile_read(self._h, ms, n.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))))
        return {p: (float(ms[i]), int(n[i])) for i, p in enumerate(PHASES)}

    # -- the two calls --
    def project_history(self, X, hist_off, stream=None) -> None:
        """Eq.(2) for every layer, once per request (RLB).  X: [T x d] rows, chronological."""
        off = _i64(hist_off)
        B = off.shape[0] - 1
        T = int(X.shape[0])
        self._check(lib().stca_project_history(self._h, ctypes.c_void_p(_ptr(X)), T,
                                                off.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), B,
                                                ctypes.c_void_p(_stream(stream))))
        self._B = B
        self._T2 = None

    def attention_backward(self, layer: int, U, dY, tgt_off, dXt=None, dU=None, stream=None):
        """stca_attention_backward (NEXT-1, partial): (dXt [T' x d], dU [N_t h x d]) float32 CUDA tensors for
        layer `layer` of the last projection, given its U (bf16 / int16 CUDA [N_t h x d]) and dY (float32)."""
        import torch
        off = _i64(tgt_off)
        B = off.shape[0] - 1
        if dXt is None:
            dXt = torch.empty((self._cache_rows(), self.d), dtype=torch.float32, device=dY.device)
        if dU is None:
            dU = torch.empty_like(dY)
        self._check(lib().stca_attention_backward(self._h, int(layer), ctypes.c_void_p(_ptr(U)), ctypes.c_void_p(_ptr(dY)),
                                                  off.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), B,
                                                  ctypes.c_void_p(_ptr(dXt)), ctypes.c_void_p(_ptr(dU)),
                                                  ctypes.c_void_p(_stream(stream))))
        return dXt, dU

    def history_backward(self, layer: int, X, dXt, dX=None, stream=None):
        """stca_history_backward (NEXT-1, partial): accumulates dX (float32 CUDA [rows x d]; zeros if None) and
        returns (dX, {"Wu", "Wv", "Wo", "ln_g", "ln_b"} weight gradients, float32 CUDA) for layer `layer`."""
        import torch
        rows = int(X.shape[0])
        rd = self.r * self.d
        if dX is None:
            dX = torch.zeros((rows, self.d), dtype=torch.float32, device=dXt.device)
        g = {"Wu": torch.empty((self.d, rd), device=dXt.device), "Wv": torch.empty((self.d, rd), device=dXt.device),
             "Wo": torch.empty((rd, self.d), device=dXt.device), "ln_g": torch.empty(self.d, device=dXt.device),
             "ln_b": torch.empty(self.d, device=dXt.device)}
        self._check(lib().stca_history_backward(self._h, int(layer), _ptr(X), rows, _ptr(dXt), _ptr(dX), _ptr(g["Wu"]),
                                                _ptr(g["Wv"]), _ptr(g["Wo"]), _ptr(g["ln_g"]), _ptr(g["ln_b"]),
                                                _stream(stream)))
        return dX, g

    def backward(self, xt, tgt_off, X, dZ, dz=None, grads=None, dX=None, dxt=None, out_Z=None, stream=None):
        """stca_backward (NEXT-1): forward over x_t, then d(sum(dZ Z_H) + sum(dz z)) for every weight role in
        `grads` (name -> float32 CUDA tensor shaped like the weight; None: all roles, allocated here), the kept
        history rows X (dX) and x_t (dxt).  Returns (grads, dX, dxt)."""
        import torch
        off = _i64(tgt_off)
        B = off.shape[0] - 1
        Nt, rows = int(xt.shape[0]), int(X.shape[0])
        dev = dZ.device
        if grads is None:
            grads = {n: torch.empty(tuple(sh), dtype=torch.float32, device=dev) for n, sh in self._shapes.items()}
        if dX is None:
            dX = torch.empty((rows, self.d), dtype=torch.float32, device=dev)
        if dxt is None:
            dxt = torch.empty((Nt, self.d), dtype=torch.float32, device=dev)
        keep = [n.encode() for n in grads]
        arr = (_Grad * max(len(grads), 1))()
        for i, (n, t) in enumerate(grads.items()):
            arr[i] = _Grad(keep[i], _ptr(t))
        self._check(lib().stca_backward(self._h, _ptr(xt), Nt, off.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), B,
                                        _ptr(X), rows, _ptr(dZ), _ptr(dz) if dz is not None else None, arr,
                                        len(grads), _ptr(dX), _ptr(dxt), _ptr(out_Z) if out_Z is not None else None,
                                        _stream(stream)))
        return grads, dX, dxt

    def _cache_rows(self) -> int:
        if getattr(self, "_T2", None) is None:
            raise ValueError("pass dXt (the cache holds sum_b L'_b rows) or call project_history with track=True")
        return self._T2

    def session_open(self, capacity_rows: int, stream=None) -> None:
        """Persistent per-user X~ cache (NEXT-4); see stca_session_open."""
        self._check(lib().stca_session_open(self._h, int(capacity_rows), ctypes.c_void_p(_stream(stream))))

    def project_history_session(self, user_id, gen, X, hist_off, stream=None) -> int:
        """stca_project_history_session: projects only users not cached with the same generation; returns the
        number of users projected."""
        off = _i64(hist_off)
        B = off.shape[0] - 1
        u, g = _i64(user_id), _i64(gen)
        if u.shape[0] != B or g.shape[0] != B:
            raise ValueError("user_id / gen need one entry per request")
        n = ctypes.c_int64(0)
        p64 = ctypes.POINTER(ctypes.c_int64)
        self._check(lib().stca_project_history_session(self._h, u.ctypes.data_as(p64), g.ctypes.data_as(p64),
                                                        ctypes.c_void_p(_ptr(X)), int(X.shape[0]),
                                                        off.ctypes.data_as(p64), B, ctypes.byref(n),
                                                        ctypes.c_void_p(_stream(stream))))
        self._B = B
        return int(n.value)

    def read_cache(self, layer: int, row0: int = 0, nrows: Optional[int] = None, out=None, stream=None):
        """Rows of the projected X~(layer) cache (compacted order) as float32; returns `out` (a new host
        array [nrows, d] unless a device or host buffer is given)."""
        if nrows is None:
            raise ValueError("nrows is required (the cache holds sum_b L'_b rows)")
        if out is None:
            out = np.empty((nrows, self.d), dtype=np.float32)
        self._check(lib().stca_read_cache(self._h, int(layer), int(row0), int(nrows), ctypes.c_void_p(_ptr(out)),
                                          ctypes.c_void_p(_stream(stream))))
        return out

    def forward(self, xt, tgt_off, out_Z, out_z=None, stream=None, sync=None) -> None:
        """Eq.(3)-(9) for the targets of the projected requests; writes out_Z [Nt,M,d], out_z [Nt,d].

        The C call only enqueues work on `stream`.  With host (numpy) outputs the binding waits for the
        stream before returning unless sync=False (then the caller synchronises, e.g. with pinned torch
        CPU tensors in a pipelined serving loop)."""
        off = _i64(tgt_off)
        B = off.shape[0] - 1
        Nt = int(xt.shape[0])
        self._check(lib().stca_forward(self._h, ctypes.c_void_p(_ptr(xt)), Nt,
                                       off.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), B,
                                       ctypes.c_void_p(_ptr(out_Z)), ctypes.c_void_p(_ptr(out_z)),
                                       ctypes.c_void_p(_stream(stream))))
        host_out = any(o is not None and not _is_cuda(o) for o in (out_Z, out_z))
        if sync or (sync is None and host_out):
            _synchronize(stream)


# ---------------------------------------------------------------------------
# split-history exchange callbacks (stca_exchange_fn): an all-gather of raw device bytes
# ---------------------------------------------------------------------------
class _DevBytes:
    """Zero-copy view of `n` device bytes at `ptr` (for torch.as_tensor)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "|u1", "data": (ptr, False), "version": 3,
                                         "strides": None}


def _torch_stream(stream: int):
    import torch
    return torch.cuda.ExternalStream(stream) if stream else torch.cuda.default_stream()


def nccl_exchange(group=None):
    """Exchange over torch.distributed (backend "nccl"): all_gather_into_tensor, ordered on the
    library's stream.  Pass as STCA(..., split_world=W, split_rank=r, exchange=nccl_exchange())."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)

    def fn(ctx, send, recv, nbytes, stream):
        try:
            s = torch.as_tensor(_DevBytes(send, nbytes), device="cuda")
            r = torch.as_tensor(_DevBytes(recv, nbytes * world), device="cuda")
            with torch.cuda.stream(_torch_stream(stream)):
                dist.all_gather_into_tensor(r, s, group=group)
            return 0
        except Exception:  # pragma: no cover
            import traceback
            traceback.print_exc()
            return 1
    return fn


class ThreadExchange:
    """G split-history ranks as host threads sharing one device (tests / emulation): the
    all-gather is done with device-to-device copies between the ranks' buffers."""

    def __init__(self, G: int):
        import threading
        self.G = G
        self.barrier = threading.Barrier(G)
        self.sends = [None] * G

    def for_rank(self, rank: int):
        import torch

        def fn(ctx, send, recv, nbytes, stream):
            try:
                st = _torch_stream(stream)
                st.synchronize()                      # this rank's partials are complete
                self.sends[rank] = (send, nbytes)
                self.barrier.wait()
                r = torch.as_tensor(_DevBytes(recv, nbytes * self.G), device="cuda")
                with torch.cuda.stream(st):
                    for g, (p, n) in enumerate(self.sends):
                        r[g * n:(g + 1) * n].copy_(torch.as_tensor(_DevBytes(p, n), device="cuda"))
                st.synchronize()
                self.barrier.wait()                   # every rank has read every send buffer
                return 0
            except Exception:  # pragma: no cover
                import traceback
                traceback.print_exc()
                return 1
        return fn


def rlb_allocate(s, hist_off, L_min: int, L_max: int, L_avg: int, stream=None):
    """stca_rlb_allocate (include/stca.h): s float64 [B], hist_off int64 [B+1], CUDA tensors.
    Returns (alloc int64 [B], new_off int64 [B+1]) as CUDA tensors."""
    import torch
    B = int(s.shape[0])
    alloc = torch.empty(B, dtype=torch.int64, device=s.device)
    new_off = torch.empty(B + 1, dtype=torch.int64, device=s.device)
    st = lib().stca_rlb_allocate(_ptr(s), _ptr(hist_off), B, int(L_min), int(L_max), int(L_avg), _ptr(alloc),
                                 _ptr(new_off), _stream(stream))
    if st != 0:
        raise StcaError(st, "stca_rlb_allocate")
    return alloc, new_off


def rlb_compact(X, hist_off, alloc, new_off, L_avg: int, P=None, stream=None):
    """stca_rlb_compact (include/stca.h): X CUDA tensor [T x d] (any 2-D dtype, rows of a
    multiple of 16 bytes).  Returns (P [B*L_avg x d] with rows < new_off[B] written, seg_off [B+1],
    segs [2B x 3]) as CUDA tensors; the number of valid triples is seg_off[B]."""
    import torch
    B = int(alloc.shape[0])
    if P is None:
        P = torch.empty((B * int(L_avg), X.shape[1]), dtype=X.dtype, device=X.device)
    seg_off = torch.empty(B + 1, dtype=torch.int64, device=X.device)
    segs = torch.empty((2 * B, 3), dtype=torch.int64, device=X.device)
    row_bytes = X.shape[1] * X.element_size()
    st = lib().stca_rlb_compact(_ptr(X), row_bytes, _ptr(hist_off), _ptr(alloc), _ptr(new_off), B, int(L_avg),
                                _ptr(P), _ptr(seg_off), _ptr(segs), _stream(stream))
    if st != 0:
        raise StcaError(st, "stca_rlb_compact")
    return P, seg_off, segs


def encode_history(video, action, position, video_id, action_id, hist_off, tdelta=None, timestamp=None,
                   req_time=None, X=None, stream=None):
    """stca_encode_history (include/stca.h): X [T x d] from ids.  Tables: CUDA tensors
    (bf16 as int16 bit patterns, or float32), video [V+1 x d] / action [A+1 x d] with the OOV row last,
    position [P x d], tdelta [NB x d] or None; ids / timestamps int64 [T], hist_off int64 [B+1],
    req_time int64 [B] (CUDA).  Returns X (same dtype as the tables)."""
    import torch
    d = int(video.shape[1])
    bf16 = video.dtype in (torch.int16, torch.bfloat16)
    T = int(video_id.shape[0])
    B = int(hist_off.shape[0]) - 1
    if X is None:
        X = torch.empty((T, d), dtype=video.dtype, device=video.device)
    tab = _EmbedTables(_ptr(video), int(video.shape[0]) - 1, _ptr(action), int(action.shape[0]) - 1,
                       _ptr(position), int(position.shape[0]), _ptr(tdelta) if tdelta is not None else None,
                       int(tdelta.shape[0]) if tdelta is not None else 0)
    st = lib().stca_encode_history(ctypes.byref(tab), d, STCA_BF16 if bf16 else STCA_FP32, _ptr(video_id),
                                   _ptr(action_id), _ptr(timestamp), _ptr(hist_off), _ptr(req_time), B, T,
                                   _ptr(X), _stream(stream))
    if st != 0:
        raise StcaError(st, "stca_encode_history")
    return X
