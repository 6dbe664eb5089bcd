"""sigb200 -- B200-native (sm_100a) signature / logsignature transforms (Signatory, arXiv 2001.00706).

Thin Python binding of libsig.so (include/sig.h).  This module only marshals arguments: it checks
that tensors are contiguous float32 CUDA tensors, allocates outputs and workspaces with PyTorch,
and passes raw device pointers plus the current CUDA stream through ctypes.  Every step of the
computation runs in the library's CUDA kernels; there is no CPU fallback -- importing works
anywhere, but any call without the built library or without a CUDA device raises.

Two layers:
  * ``sig_*`` functions with the same names and argument order as the C ABI (no autograd);
  * differentiable ``signature``, ``logsignature``, ``signature_combine``,
    ``multi_signature_combine`` (torch.autograd.Function wrappers whose backward calls the
    handwritten reversible backward kernels).
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np
import torch

__all__ = [
    "lib", "LIB_PATH", "SigError",
    "sig_signature_channels", "sig_logsignature_channels", "sig_is_supported",
    "sig_signature", "sig_signature_backward", "sig_signature_save", "sig_signature_backward_saved",
    "sig_signature_combine", "sig_signature_combine_backward",
    "sig_multi_signature_combine", "LogSigPlan", "sig_logsignature", "sig_logsignature_backward",
    "signature", "logsignature", "signature_combine", "multi_signature_combine",
    "BP_NONE", "BP_ZERO", "BP_GIVEN", "MODES",
]

# SIGB200_LIB may point at an alternative build of the same library (A/B experiments)
LIB_PATH = os.environ.get("SIGB200_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsig.so")
BP_NONE, BP_ZERO, BP_GIVEN = 0, 1, 2
MODES = {"expand": 0, "brackets": 1, "words": 2}

_c_i64, _c_i32, _c_sz, _vp = ctypes.c_int64, ctypes.c_int32, ctypes.c_size_t, ctypes.c_void_p


class SigError(RuntimeError):
    pass


_lib = None
_lock = threading.Lock()


def lib():
    """Load libsig.so (build it with ``python -m paper_2001_00706_b200.build``).  Raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise SigError(f"{LIB_PATH} is missing: build it with `python -m paper_2001_00706_b200.build` "
                               "(there is no CPU fallback)")
            L = ctypes.CDLL(LIB_PATH)
            sig = [
                ("sig_signature_channels", _c_i64, [_c_i64, _c_i32]),
                ("sig_logsignature_channels", _c_i64, [_c_i64, _c_i32, ctypes.c_int]),
                ("sig_is_supported", _c_i32, [_c_i64, _c_i32, _c_i32]),
                ("sig_status_string", ctypes.c_char_p, [ctypes.c_int]),
                ("sig_launch_count", ctypes.c_uint64, []),
                ("sig_last_error", ctypes.c_char_p, []),
                ("sig_signature_workspace_size", _c_sz, [_c_i64, _c_i64, _c_i64, _c_i32, _c_i32, ctypes.c_int]),
                ("sig_signature", ctypes.c_int, [_vp, _c_i64, _c_i64, _c_i64, _c_i32, _c_i32, ctypes.c_int, _vp, _vp,
                                                 _vp, _c_sz, _vp]),
                ("sig_signature_backward", ctypes.c_int, [_vp, _vp, _vp, _c_i64, _c_i64, _c_i64, _c_i32, _c_i32,
                                                          ctypes.c_int, _vp, _vp, _vp, _vp]),
                ("sig_signature_ex_workspace_size", _c_sz, [_c_i64, _c_i64, _c_i64, _c_i32, _c_i32, ctypes.c_int,
                                                            _c_i32, _c_i32]),
                ("sig_signature_ex", ctypes.c_int, [_vp, _c_i64, _c_i64, _c_i64, _c_i32, _c_i32, ctypes.c_int, _vp,
                                                    _c_i32, _vp, _vp, _vp, _c_sz, _vp]),
                ("sig_signature_backward_ex_workspace_size", _c_sz, [_c_i64, _c_i64, _c_i64, _c_i32, _c_i32,
                                                                     ctypes.c_int, _c_i32, _c_i32, _c_i32]),
                ("sig_signature_backward_ex", ctypes.c_int, [_vp, _vp, _vp, _c_i64, _c_i64, _c_i64, _c_i32, _c_i32,
                                                             ctypes.c_int, _vp, _c_i32, _vp, _vp, _vp, _vp, _vp,
                                                             _c_sz, _vp]),
                ("sig_signature_saved_bytes", _c_sz, [_c_i64, _c_i64, _c_i64, _c_i32, ctypes.c_int]),
                ("sig_signature_save_workspace_size", _c_sz, [_c_i64, _c_i64, _c_i64, _c_i32, ctypes.c_int]),
                ("sig_signature_save", ctypes.c_int, [_vp, _c_i64, _c_i64, _c_i64, _c_i32, ctypes.c_int, _vp, _vp,
                                                      _vp, _c_sz, _vp, _c_sz, _vp]),
                ("sig_signature_backward_saved_workspace_size", _c_sz, [_c_i64, _c_i64, _c_i64, _c_i32,
                                                                        ctypes.c_int]),
                ("sig_signature_backward_saved", ctypes.c_int, [_vp, _vp, _vp, _vp, _c_sz, _c_i64, _c_i64, _c_i64,
                                                                _c_i32, ctypes.c_int, _vp, _vp, _vp, _vp, _c_sz,
                                                                _vp]),
                ("sig_signature_fwd_bwd_host_workspace_size", _c_sz, [_c_i64, _c_i64, _c_i64, _c_i32, _c_i32]),
                ("sig_signature_fwd_bwd_host", ctypes.c_int, [_vp, _vp, _c_i64, _c_i64, _c_i64, _c_i32, _vp, _c_i32,
                                                              _vp, _c_sz, _vp]),
                ("sig_signature_combine", ctypes.c_int, [_vp, _vp, _c_i64, _c_i64, _c_i32, _vp, _vp]),
                ("sig_signature_combine_backward", ctypes.c_int, [_vp, _vp, _vp, _c_i64, _c_i64, _c_i32, _vp, _vp,
                                                                  _vp]),
                ("sig_multi_signature_combine_workspace_size", _c_sz, [_c_i64, _c_i64, _c_i64, _c_i32]),
                ("sig_multi_signature_combine", ctypes.c_int, [_vp, _c_i64, _c_i64, _c_i64, _c_i32, _vp, _vp, _c_sz,
                                                               _vp]),
                ("sig_logsig_plan_create", ctypes.c_int, [_c_i64, _c_i32, ctypes.c_int, ctypes.POINTER(_vp)]),
                ("sig_logsig_plan_destroy", ctypes.c_int, [_vp]),
                ("sig_logsignature_workspace_size", _c_sz, [_vp, _c_i64, _c_i64, _c_i32, ctypes.c_int]),
                ("sig_logsignature", ctypes.c_int, [_vp, _vp, _c_i64, _c_i64, _c_i32, ctypes.c_int, _vp, _vp, _vp,
                                                    _vp, _c_sz, _vp]),
                ("sig_logsignature_backward", ctypes.c_int, [_vp, _vp, _vp, _vp, _c_i64, _c_i64, _c_i32, ctypes.c_int,
                                                             _vp, _vp, _vp, _vp, _c_sz, _vp]),
                ("sig_logsignature_from_signature_workspace_size", _c_sz, [_vp, _c_i64]),
                ("sig_logsignature_from_signature", ctypes.c_int, [_vp, _vp, _c_i64, _vp, _vp]),
                ("sig_logsignature_from_signature_backward", ctypes.c_int, [_vp, _vp, _vp, _c_i64, _vp, _vp, _c_sz,
                                                                            _vp]),
                ("sig_path_query_workspace_size", _c_sz, [_c_i64, _c_i64]),
                ("sig_path_query", ctypes.c_int, [_vp, _vp, _c_i64, _c_i64, _c_i64, _c_i32, _vp, _vp, _c_i64, _vp,
                                                  _vp, _c_sz, _vp]),
                ("sig_path_query_backward", ctypes.c_int, [_vp, _vp, _vp, _c_i64, _c_i64, _c_i64, _c_i32, _vp, _vp,
                                                           _c_i64, _vp, _vp, _vp, _c_sz, _vp]),
            ]
            for name, res, args in sig:
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def _on_device(fn):
    """Run a C-ABI mirror with the CUDA device of its first CUDA tensor argument current: the library
    launches on the current device, and the stream passed is that tensor's device stream."""
    import functools

    @functools.wraps(fn)
    def wrapped(*args, **kwargs):
        for a in list(args) + list(kwargs.values()):
            if isinstance(a, torch.Tensor) and a.is_cuda:
                with torch.cuda.device(a.device):
                    return fn(*args, **kwargs)
        return fn(*args, **kwargs)

    return wrapped


def _shape(t: torch.Tensor, want: tuple, name: str):
    if tuple(t.shape) != tuple(want):
        raise SigError(f"{name} must have shape {list(want)}, got {list(t.shape)}")


def _path3(path: torch.Tensor):
    if path.dim() != 3:
        raise SigError(f"path must be [B, L, C], got shape {list(path.shape)}")
    return path.shape


def _check(status: int, what: str):
    if status != 0:
        L = lib()
        raise SigError(f"{what}: {L.sig_status_string(status).decode()}: {L.sig_last_error().decode()}")


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(device) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _dev_f32(t: torch.Tensor, name: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if not t.is_cuda:
        raise SigError(f"{name} must be a CUDA tensor (sm_100a kernels only; no CPU fallback)")
    if t.dtype != torch.float32:
        raise TypeError(f"{name} must be float32, got {t.dtype}")
    return t.contiguous()


def _bp(basepoint, path):
    """basepoint: None/False -> NONE; True -> ZERO; tensor [B, C] -> GIVEN (reading R4)."""
    if basepoint is None or basepoint is False:
        return BP_NONE, None
    if basepoint is True:
        return BP_ZERO, None
    bp = _dev_f32(basepoint, "basepoint")
    B, C = path.shape[0], path.shape[-1]
    if bp.dim() == 1:
        bp = bp.unsqueeze(0)
    if bp.dim() != 2 or bp.shape[-1] != C or bp.shape[0] not in (1, B):
        raise SigError(f"basepoint must be [{C}], [1, {C}] or [{B}, {C}], got {list(basepoint.shape)}")
    if bp.shape[0] != B:
        bp = bp.expand(B, -1).contiguous()
    return BP_GIVEN, bp


# ------------------------------------------------------------------------------------------------
# C-ABI mirrors
# ------------------------------------------------------------------------------------------------
def sig_signature_channels(C: int, depth: int) -> int:
    return int(lib().sig_signature_channels(C, depth))


def sig_logsignature_channels(C: int, depth: int, mode: str = "words") -> int:
    return int(lib().sig_logsignature_channels(C, depth, MODES[mode]))


def sig_is_supported(C: int, depth: int, backward: bool = False) -> bool:
    return bool(lib().sig_is_supported(C, depth, int(backward)))


@_on_device
def sig_signature(path: torch.Tensor, depth: int, stream: bool = False, basepoint=None, inverse: bool = False,
                  initial=None) -> torch.Tensor:
    """sig_signature / sig_signature_ex: inverse and initial as in include/sig.h (reading R18)."""
    path = _dev_f32(path, "path")
    B, L, C = _path3(path)
    bpm, bp = _bp(basepoint, path)
    Lib = lib()
    S = Lib.sig_signature_channels(C, depth)
    if S < 0:
        raise SigError(f"bad C={C} depth={depth}")
    if initial is not None:
        _shape(initial, (B, S), "initial")
    M = L - 1 + (bpm != BP_NONE)
    out = torch.empty((B, M, S) if stream else (B, S), device=path.device, dtype=torch.float32)
    if not inverse and initial is None:
        wsb = Lib.sig_signature_workspace_size(B, L, C, depth, int(stream), bpm)
        ws = torch.empty(wsb, device=path.device, dtype=torch.uint8) if wsb else None
        _check(Lib.sig_signature(_ptr(path), B, L, C, depth, int(stream), bpm, _ptr(bp), _ptr(out), _ptr(ws), wsb,
                                 _stream(path.device)), "sig_signature")
        return out
    ini = None if initial is None else _dev_f32(initial, "initial")
    wsb = Lib.sig_signature_ex_workspace_size(B, L, C, depth, int(stream), bpm, int(inverse), int(ini is not None))
    ws = torch.empty(wsb, device=path.device, dtype=torch.uint8) if wsb else None
    _check(Lib.sig_signature_ex(_ptr(path), B, L, C, depth, int(stream), bpm, _ptr(bp), int(inverse), _ptr(ini),
                                _ptr(out), _ptr(ws), wsb, _stream(path.device)), "sig_signature_ex")
    return out


def sig_signature_backward(grad_out, path, out_saved, depth: int, stream: bool = False, basepoint=None):
    """-> (grad_path, grad_basepoint or None).  Goes through sig_signature_backward_ex with its
    full workspace, so small batches and long paths use the time-parallel (chunked) backward."""
    gp, gbp, _ = sig_signature_backward_ex(grad_out, path, out_saved, depth, stream, basepoint,
                                           want_grad_initial=False)
    return gp, gbp


@_on_device
def sig_signature_backward_ex(grad_out, path, out_saved, depth: int, stream: bool = False, basepoint=None,
                              inverse: bool = False, initial=None, want_grad_initial: bool = True):
    """-> (grad_path, grad_basepoint or None, grad_initial or None)."""
    path = _dev_f32(path, "path")
    grad_out = _dev_f32(grad_out, "grad_out")
    out_saved = _dev_f32(out_saved, "out_saved")
    B, L, C = _path3(path)
    bpm, bp = _bp(basepoint, path)
    ini = None if initial is None else _dev_f32(initial, "initial")
    Lib = lib()
    S = Lib.sig_signature_channels(C, depth)
    if S < 0:
        raise SigError(f"bad C={C} depth={depth}")
    M = L - 1 + (bpm != BP_NONE)
    want = (B, M, S) if stream else (B, S)
    _shape(grad_out, want, "grad_out")
    _shape(out_saved, want, "out_saved")
    if ini is not None:
        _shape(ini, (B, S), "initial")
    gp = torch.empty_like(path)
    gbp = torch.empty((B, C), device=path.device, dtype=torch.float32) if bpm == BP_GIVEN else None
    gi = torch.empty((B, S), device=path.device, dtype=torch.float32) if want_grad_initial else None
    wsb = Lib.sig_signature_backward_ex_workspace_size(B, L, C, depth, int(stream), bpm, int(inverse),
                                                       int(ini is not None), int(gi is not None))
    ws = torch.empty(wsb, device=path.device, dtype=torch.uint8) if wsb else None
    _check(Lib.sig_signature_backward_ex(_ptr(grad_out), _ptr(path), _ptr(out_saved), B, L, C, depth, int(stream),
                                         bpm, _ptr(bp), int(inverse), _ptr(ini), _ptr(gp), _ptr(gbp), _ptr(gi),
                                         _ptr(ws), wsb, _stream(path.device)), "sig_signature_backward_ex")
    return gp, gbp, gi


@_on_device
def sig_signature_save(path, depth: int, basepoint=None):
    """sig_signature_save: the signature plus the chunk states the time-parallel backward starts
    from (include/sig.h) -> (out [B, S], saved uint8 tensor or None when the backward would not
    chunk).  Pass both to sig_signature_backward_saved."""
    path = _dev_f32(path, "path")
    B, L, C = _path3(path)
    bpm, bp = _bp(basepoint, path)
    Lib = lib()
    S = Lib.sig_signature_channels(C, depth)
    if S < 0:
        raise SigError(f"bad C={C} depth={depth}")
    out = torch.empty((B, S), device=path.device, dtype=torch.float32)
    sb = Lib.sig_signature_saved_bytes(B, L, C, depth, bpm)
    saved = torch.empty(sb, device=path.device, dtype=torch.uint8) if sb else None
    wsb = Lib.sig_signature_save_workspace_size(B, L, C, depth, bpm)
    ws = torch.empty(wsb, device=path.device, dtype=torch.uint8) if wsb else None
    _check(Lib.sig_signature_save(_ptr(path), B, L, C, depth, bpm, _ptr(bp), _ptr(out), _ptr(saved), sb, _ptr(ws),
                                  wsb, _stream(path.device)), "sig_signature_save")
    return out, saved


@_on_device
def sig_signature_backward_saved(grad_out, path, out_saved, saved, depth: int, basepoint=None):
    """sig_signature_backward_saved -> (grad_path, grad_basepoint or None)."""
    path = _dev_f32(path, "path")
    grad_out = _dev_f32(grad_out, "grad_out")
    out_saved = _dev_f32(out_saved, "out_saved")
    B, L, C = _path3(path)
    bpm, bp = _bp(basepoint, path)
    Lib = lib()
    S = Lib.sig_signature_channels(C, depth)
    if S < 0:
        raise SigError(f"bad C={C} depth={depth}")
    _shape(grad_out, (B, S), "grad_out")
    _shape(out_saved, (B, S), "out_saved")
    sb = Lib.sig_signature_saved_bytes(B, L, C, depth, bpm)
    if sb and (saved is None or saved.numel() < sb or saved.device != path.device):
        raise SigError(f"saved must be the {sb}-byte tensor sig_signature_save returned for this call")
    gp = torch.empty_like(path)
    gbp = torch.empty((B, C), device=path.device, dtype=torch.float32) if bpm == BP_GIVEN else None
    wsb = Lib.sig_signature_backward_saved_workspace_size(B, L, C, depth, bpm)
    ws = torch.empty(wsb, device=path.device, dtype=torch.uint8) if wsb else None
    _check(Lib.sig_signature_backward_saved(_ptr(grad_out), _ptr(path), _ptr(out_saved),
                                            _ptr(saved) if sb else None, sb, B, L, C, depth, bpm, _ptr(bp),
                                            _ptr(gp), _ptr(gbp), _ptr(ws), wsb, _stream(path.device)),
           "sig_signature_backward_saved")
    return gp, gbp


def sig_signature_fwd_bwd_host(path_h, grad_out_h, depth: int, chunks: int = 4, grad_path_h=None, device=None):
    """sig_signature_fwd_bwd_host: forward + reversible backward of a HOST-resident batch, in
    `chunks` slices whose copies overlap the kernels (include/sig.h).  path_h [B, L, C] and
    grad_out_h [B, S] are float32 CPU tensors (pinned for the overlap); returns grad_path [B, L, C]
    in host memory (grad_path_h if given), valid once the current CUDA stream completes."""
    for name, t in (("path_h", path_h), ("grad_out_h", grad_out_h)):
        if t.device.type != "cpu" or t.dtype != torch.float32 or not t.is_contiguous():
            raise SigError(f"{name} must be a contiguous float32 CPU tensor")
    B, L, C = path_h.shape
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    Lib = lib()
    S = Lib.sig_signature_channels(C, depth)
    if tuple(grad_out_h.shape) != (B, S):
        raise SigError(f"grad_out_h must be [{B}, {S}]")
    out = grad_path_h if grad_path_h is not None else torch.empty((B, L, C), dtype=torch.float32).pin_memory()
    wsb = Lib.sig_signature_fwd_bwd_host_workspace_size(B, L, C, depth, chunks)
    ws = torch.empty(max(wsb, 1), device=dev, dtype=torch.uint8)
    _check(Lib.sig_signature_fwd_bwd_host(_ptr(path_h), _ptr(grad_out_h), B, L, C, depth, _ptr(out), chunks,
                                          _ptr(ws), wsb, _stream(dev)), "sig_signature_fwd_bwd_host")
    return out


@_on_device
def sig_signature_combine(a, b, C: int, depth: int):
    a, b = _dev_f32(a, "a"), _dev_f32(b, "b")
    S = sig_signature_channels(C, depth)
    if a.dim() != 2 or a.shape[1] != S:
        raise SigError(f"a must be [B, {S}], got {list(a.shape)}")
    _shape(b, tuple(a.shape), "b")
    out = torch.empty_like(a)
    _check(lib().sig_signature_combine(_ptr(a), _ptr(b), a.shape[0], C, depth, _ptr(out), _stream(a.device)),
           "sig_signature_combine")
    return out


@_on_device
def sig_signature_combine_backward(grad_out, a, b, C: int, depth: int):
    grad_out, a, b = _dev_f32(grad_out, "grad_out"), _dev_f32(a, "a"), _dev_f32(b, "b")
    S = sig_signature_channels(C, depth)
    if a.dim() != 2 or a.shape[1] != S:
        raise SigError(f"a must be [B, {S}], got {list(a.shape)}")
    _shape(b, tuple(a.shape), "b")
    _shape(grad_out, tuple(a.shape), "grad_out")
    ga, gb = torch.empty_like(a), torch.empty_like(b)
    _check(lib().sig_signature_combine_backward(_ptr(grad_out), _ptr(a), _ptr(b), a.shape[0], C, depth, _ptr(ga),
                                                _ptr(gb), _stream(a.device)), "sig_signature_combine_backward")
    return ga, gb


@_on_device
def sig_multi_signature_combine(sigs, C: int, depth: int):
    """sigs [n, B, S] in time order -> [B, S]."""
    sigs = _dev_f32(sigs, "sigs")
    if sigs.dim() != 3 or sigs.shape[2] != sig_signature_channels(C, depth):
        raise SigError(f"sigs must be [n, B, {sig_signature_channels(C, depth)}], got {list(sigs.shape)}")
    n, B, S = sigs.shape
    Lib = lib()
    out = torch.empty((B, S), device=sigs.device, dtype=torch.float32)
    wsb = Lib.sig_multi_signature_combine_workspace_size(n, B, C, depth)
    ws = torch.empty(wsb, device=sigs.device, dtype=torch.uint8) if wsb else None
    _check(Lib.sig_multi_signature_combine(_ptr(sigs), n, B, C, depth, _ptr(out), _ptr(ws), wsb,
                                           _stream(sigs.device)), "sig_multi_signature_combine")
    return out


class LogSigPlan:
    """Owns a sig_logsig_plan_t (device tables for one (C, depth, mode)), per device."""

    _cache: dict = {}

    def __init__(self, C: int, depth: int, mode: str = "words"):
        self.C, self.depth, self.mode = C, depth, mode
        self.handle = ctypes.c_void_p()
        _check(lib().sig_logsig_plan_create(C, depth, MODES[mode], ctypes.byref(self.handle)),
               "sig_logsig_plan_create")
        self.width = sig_logsignature_channels(C, depth, mode)

    def __del__(self):
        try:
            if self.handle:
                lib().sig_logsig_plan_destroy(self.handle)
        except Exception:
            pass

    @classmethod
    def get(cls, C: int, depth: int, mode: str, device) -> "LogSigPlan":
        key = (C, depth, mode, torch.device(device).index)
        if key not in cls._cache:
            with torch.cuda.device(device):
                cls._cache[key] = LogSigPlan(C, depth, mode)
        return cls._cache[key]


@_on_device
def sig_logsignature(path, depth: int, mode: str = "words", stream: bool = False, basepoint=None,
                     return_signature: bool = False):
    path = _dev_f32(path, "path")
    B, L, C = _path3(path)
    plan = LogSigPlan.get(C, depth, mode, path.device)
    bpm, bp = _bp(basepoint, path)
    Lib = lib()
    M = L - 1 + (bpm != BP_NONE)
    S = sig_signature_channels(C, depth)
    out = torch.empty((B, M, plan.width) if stream else (B, plan.width), device=path.device, dtype=torch.float32)
    sig = torch.empty((B, M, S) if stream else (B, S), device=path.device, dtype=torch.float32)
    wsb = Lib.sig_logsignature_workspace_size(plan.handle, B, L, int(stream), bpm)
    ws = torch.empty(wsb, device=path.device, dtype=torch.uint8) if wsb else None
    _check(Lib.sig_logsignature(plan.handle, _ptr(path), B, L, int(stream), bpm, _ptr(bp), _ptr(out), _ptr(sig),
                                _ptr(ws), wsb, _stream(path.device)), "sig_logsignature")
    return (out, sig) if return_signature else out


@_on_device
def sig_logsignature_backward(grad_out, path, sig_saved, depth: int, mode: str = "words", stream: bool = False,
                              basepoint=None):
    path = _dev_f32(path, "path")
    grad_out = _dev_f32(grad_out, "grad_out")
    sig_saved = _dev_f32(sig_saved, "sig_saved")
    B, L, C = _path3(path)
    plan = LogSigPlan.get(C, depth, mode, path.device)
    bpm, bp = _bp(basepoint, path)
    Lib = lib()
    M = L - 1 + (bpm != BP_NONE)
    S = sig_signature_channels(C, depth)
    _shape(grad_out, (B, M, plan.width) if stream else (B, plan.width), "grad_out")
    _shape(sig_saved, (B, M, S) if stream else (B, S), "sig_saved")
    gp = torch.empty_like(path)
    gbp = torch.empty((B, C), device=path.device, dtype=torch.float32) if bpm == BP_GIVEN else None
    wsb = Lib.sig_logsignature_workspace_size(plan.handle, B, L, int(stream), bpm)
    ws = torch.empty(wsb, device=path.device, dtype=torch.uint8) if wsb else None
    _check(Lib.sig_logsignature_backward(plan.handle, _ptr(grad_out), _ptr(path), _ptr(sig_saved), B, L, int(stream),
                                         bpm, _ptr(bp), _ptr(gp), _ptr(gbp), _ptr(ws), wsb, _stream(path.device)),
           "sig_logsignature_backward")
    return gp, gbp


# ------------------------------------------------------------------------------------------------
# differentiable API (Signatory-style)
# ------------------------------------------------------------------------------------------------
class _Signature(torch.autograd.Function):
    @staticmethod
    def forward(ctx, path, depth, stream, basepoint_flag, bp_tensor, inverse, initial, save):
        # save: a backward will follow (grad mode on and path requires grad, decided by the caller:
        # inside forward grad mode is always off)
        bp = bp_tensor if basepoint_flag == BP_GIVEN else (basepoint_flag == BP_ZERO)
        ctx.chunks = None
        if save and not stream and not inverse and initial is None:
            # a backward will follow: keep the chunk states its time-parallel reversal starts from
            # (None when the batch fills the GPU without chunks)
            out, ctx.chunks = sig_signature_save(path, depth, bp)
        else:
            out = sig_signature(path, depth, stream, bp, inverse=inverse, initial=initial)
        ctx.save_for_backward(path, out, bp_tensor if basepoint_flag == BP_GIVEN else None, initial)
        ctx.depth, ctx.stream, ctx.bpf, ctx.inverse = depth, stream, basepoint_flag, inverse
        return out

    @staticmethod
    def backward(ctx, grad_out):
        path, out, bpt, initial = ctx.saved_tensors
        bp = bpt if ctx.bpf == BP_GIVEN else (ctx.bpf == BP_ZERO)
        if ctx.chunks is not None:
            gp, gbp = sig_signature_backward_saved(grad_out.contiguous(), path, out, ctx.chunks, ctx.depth, bp)
            ctx.chunks = None
            return gp, None, None, None, gbp, None, None, None
        if not ctx.inverse and initial is None:
            gp, gbp = sig_signature_backward(grad_out.contiguous(), path, out, ctx.depth, ctx.stream, bp)
            return gp, None, None, None, gbp, None, None, None
        gp, gbp, gi = sig_signature_backward_ex(grad_out.contiguous(), path, out, ctx.depth, ctx.stream, bp,
                                                inverse=ctx.inverse, initial=initial,
                                                want_grad_initial=initial is not None and ctx.needs_input_grad[6])
        return gp, None, None, None, gbp, None, gi, None


def _bp_args(basepoint):
    if basepoint is None or basepoint is False:
        return BP_NONE, None
    if basepoint is True:
        return BP_ZERO, None
    return BP_GIVEN, basepoint


def signature(path: torch.Tensor, depth: int, stream: bool = False, basepoint=None, inverse: bool = False,
              initial=None) -> torch.Tensor:
    """Sig^depth of each stream in path [B, L, C] -> [B, S] (or [B, M, S] with stream=True).
    inverse: Sig(x)^{-1} = Sig(x reversed); initial [B, S]: the update case
     -- initial [x] Sig, or Sig^{-1} [x] initial with inverse (reading R18).
    Differentiable in path, basepoint and initial; the backward is the reversible kernel."""
    f, t = _bp_args(basepoint)
    save = torch.is_grad_enabled() and path.requires_grad
    return _Signature.apply(path, depth, stream, f, t, bool(inverse), initial, save)


class _LogSignature(torch.autograd.Function):
    @staticmethod
    def forward(ctx, path, depth, mode, stream, basepoint_flag, bp_tensor):
        bp = bp_tensor if basepoint_flag == BP_GIVEN else (basepoint_flag == BP_ZERO)
        out, sig = sig_logsignature(path, depth, mode, stream, bp, return_signature=True)
        ctx.save_for_backward(path, sig, bp_tensor if basepoint_flag == BP_GIVEN else None)
        ctx.depth, ctx.mode, ctx.stream, ctx.bpf = depth, mode, stream, basepoint_flag
        return out

    @staticmethod
    def backward(ctx, grad_out):
        path, sig, bpt = ctx.saved_tensors
        bp = bpt if ctx.bpf == BP_GIVEN else (ctx.bpf == BP_ZERO)
        gp, gbp = sig_logsignature_backward(grad_out.contiguous(), path, sig, ctx.depth, ctx.mode, ctx.stream, bp)
        return gp, None, None, None, None, gbp


def logsignature(path: torch.Tensor, depth: int, mode: str = "words", stream: bool = False,
                 basepoint=None, inverse: bool = False) -> torch.Tensor:
    """LogSig^depth in the 'words' (default), 'brackets' or 'expand' basis.
    inverse: the logsignature of the inverted signature (of every prefix with
    stream=True) -- the inverse signature scan (K1) followed by K4, both differentiable."""
    if inverse:
        sig = signature(path, depth, stream=stream, basepoint=basepoint, inverse=True)
        return signature_to_logsignature(sig, path.shape[-1], depth, mode)
    f, t = _bp_args(basepoint)
    return _LogSignature.apply(path, depth, mode, stream, f, t)


class _Combine(torch.autograd.Function):
    @staticmethod
    def forward(ctx, a, b, C, depth):
        ctx.save_for_backward(a, b)
        ctx.C, ctx.depth = C, depth
        return sig_signature_combine(a, b, C, depth)

    @staticmethod
    def backward(ctx, g):
        a, b = ctx.saved_tensors
        ga, gb = sig_signature_combine_backward(g.contiguous(), a, b, ctx.C, ctx.depth)
        return ga, gb, None, None


def signature_combine(a: torch.Tensor, b: torch.Tensor, C: int, depth: int) -> torch.Tensor:
    """a [x] b (Chen's identity), differentiable."""
    return _Combine.apply(a, b, C, depth)


def multi_signature_combine(sigs, C: int, depth: int) -> torch.Tensor:
    """Ordered product of a list / [n, B, S] stack of signatures (forward only)."""
    if isinstance(sigs, (list, tuple)):
        sigs = torch.stack(list(sigs))
    return sig_multi_signature_combine(sigs, C, depth)


# ------------------------------------------------------------------------------------------------
# logsignature of given signatures, and Path
# ------------------------------------------------------------------------------------------------
@_on_device
def sig_logsignature_from_signature(sig, C: int, depth: int, mode: str = "words"):
    sig = _dev_f32(sig, "sig")
    S = sig_signature_channels(C, depth)
    if sig.shape[-1] != S:
        raise SigError(f"sig must be [..., {S}], got {list(sig.shape)}")
    rows = sig.numel() // S
    plan = LogSigPlan.get(C, depth, mode, sig.device)
    out = torch.empty(tuple(sig.shape[:-1]) + (plan.width,), device=sig.device, dtype=torch.float32)
    _check(lib().sig_logsignature_from_signature(plan.handle, _ptr(sig), rows, _ptr(out), _stream(sig.device)),
           "sig_logsignature_from_signature")
    return out


@_on_device
def sig_logsignature_from_signature_backward(grad_out, sig, C: int, depth: int, mode: str = "words"):
    sig = _dev_f32(sig, "sig")
    grad_out = _dev_f32(grad_out, "grad_out")
    S = sig_signature_channels(C, depth)
    if sig.shape[-1] != S:
        raise SigError(f"sig must be [..., {S}], got {list(sig.shape)}")
    _shape(grad_out, tuple(sig.shape[:-1]) + (sig_logsignature_channels(C, depth, mode),), "grad_out")
    rows = sig.numel() // S
    plan = LogSigPlan.get(C, depth, mode, sig.device)
    Lib = lib()
    wsb = Lib.sig_logsignature_from_signature_workspace_size(plan.handle, rows)
    ws = torch.empty(wsb, device=sig.device, dtype=torch.uint8) if wsb else None
    gs = torch.empty_like(sig)
    _check(Lib.sig_logsignature_from_signature_backward(plan.handle, _ptr(grad_out), _ptr(sig), rows, _ptr(gs),
                                                        _ptr(ws), wsb, _stream(sig.device)),
           "sig_logsignature_from_signature_backward")
    return gs


class _SigToLogsig(torch.autograd.Function):
    @staticmethod
    def forward(ctx, sig, C, depth, mode):
        ctx.save_for_backward(sig)
        ctx.C, ctx.depth, ctx.mode = C, depth, mode
        return sig_logsignature_from_signature(sig, C, depth, mode)

    @staticmethod
    def backward(ctx, grad_out):
        (sig,) = ctx.saved_tensors
        return sig_logsignature_from_signature_backward(grad_out.contiguous(), sig, ctx.C, ctx.depth, ctx.mode), \
            None, None, None


def signature_to_logsignature(sig, C: int, depth: int, mode: str = "words"):
    """Logsignature of given signature rows [..., S] (K4; differentiable through K5)."""
    return _SigToLogsig.apply(sig, C, depth, mode)


def _queries(starts, ends):
    qs = np.ascontiguousarray(np.asarray(starts, dtype=np.int64).reshape(-1))
    qe = np.ascontiguousarray(np.asarray(ends, dtype=np.int64).reshape(-1))
    if qs.shape != qe.shape:
        raise ValueError("starts and ends must have the same length")
    return qs, qe


@_on_device
def sig_path_query(prefix_sig, prefix_inv, C: int, depth: int, starts, ends):
    prefix_sig = _dev_f32(prefix_sig, "prefix_sig")
    prefix_inv = _dev_f32(prefix_inv, "prefix_inv")
    if prefix_sig.dim() != 3 or prefix_sig.shape[2] != sig_signature_channels(C, depth):
        raise SigError(f"prefix_sig must be [B, M, {sig_signature_channels(C, depth)}], got {list(prefix_sig.shape)}")
    _shape(prefix_inv, tuple(prefix_sig.shape), "prefix_inv")
    B, M, S = prefix_sig.shape
    qs, qe = _queries(starts, ends)
    Q = qs.shape[0]
    Lib = lib()
    out = torch.empty((B, Q, S), device=prefix_sig.device, dtype=torch.float32)
    wsb = Lib.sig_path_query_workspace_size(M, Q)
    ws = torch.empty(wsb, device=prefix_sig.device, dtype=torch.uint8) if wsb else None
    _check(Lib.sig_path_query(_ptr(prefix_sig), _ptr(prefix_inv), B, M, C, depth, qs.ctypes.data_as(_vp),
                              qe.ctypes.data_as(_vp), Q, _ptr(out), _ptr(ws), wsb, _stream(prefix_sig.device)),
           "sig_path_query")
    return out


@_on_device
def sig_path_query_backward(grad_out, prefix_sig, prefix_inv, C: int, depth: int, starts, ends):
    prefix_sig = _dev_f32(prefix_sig, "prefix_sig")
    prefix_inv = _dev_f32(prefix_inv, "prefix_inv")
    grad_out = _dev_f32(grad_out, "grad_out")
    if prefix_sig.dim() != 3 or prefix_sig.shape[2] != sig_signature_channels(C, depth):
        raise SigError(f"prefix_sig must be [B, M, {sig_signature_channels(C, depth)}], got {list(prefix_sig.shape)}")
    _shape(prefix_inv, tuple(prefix_sig.shape), "prefix_inv")
    B, M, S = prefix_sig.shape
    qs, qe = _queries(starts, ends)
    Q = qs.shape[0]
    _shape(grad_out, (B, Q, S), "grad_out")
    Lib = lib()
    gs = torch.empty_like(prefix_sig)
    gi = torch.empty_like(prefix_inv)
    wsb = Lib.sig_path_query_workspace_size(M, Q)
    ws = torch.empty(wsb, device=prefix_sig.device, dtype=torch.uint8) if wsb else None
    _check(Lib.sig_path_query_backward(_ptr(grad_out), _ptr(prefix_sig), _ptr(prefix_inv), B, M, C, depth,
                                       qs.ctypes.data_as(_vp), qe.ctypes.data_as(_vp), Q, _ptr(gs), _ptr(gi),
                                       _ptr(ws), wsb, _stream(prefix_sig.device)), "sig_path_query_backward")
    return gs, gi


class _PathQuery(torch.autograd.Function):
    @staticmethod
    def forward(ctx, prefix_sig, prefix_inv, C, depth, starts, ends):
        ctx.save_for_backward(prefix_sig, prefix_inv)
        ctx.C, ctx.depth, ctx.starts, ctx.ends = C, depth, starts, ends
        return sig_path_query(prefix_sig, prefix_inv, C, depth, starts, ends)

    @staticmethod
    def backward(ctx, grad_out):
        ps, pi = ctx.saved_tensors
        gs, gi = sig_path_query_backward(grad_out.contiguous(), ps, pi, ctx.C, ctx.depth, ctx.starts, ctx.ends)
        return gs, gi, None, None, None, None


class Path:
    """Signatory's Path: O(L) precomputation -- the prefix signatures and prefix
    inverse signatures of the stream (K1, stream mode) -- then any interval's signature in O(1)
    by one [x] (sig_path_query), its logsignature by a log of that (K4), and `update` to append
    new points (the initial option).  Differentiable w.r.t. the path (and basepoint).

    Indices follow Python slicing over the (augmented, if a basepoint is given) points:
    signature(start, end) = Sig(x[start:end]), end - start >= 2."""

    def __init__(self, path: torch.Tensor, depth: int, basepoint=None):
        if path.dim() != 3:
            raise ValueError("path must be [B, L, C]")
        self.depth = depth
        self.channels = path.shape[-1]
        self._sig = signature(path, depth, stream=True, basepoint=basepoint)
        self._inv = signature(path, depth, stream=True, basepoint=basepoint, inverse=True)
        self._last = path[:, -1, :]
        self._npoints = path.shape[1] + (0 if basepoint is None or basepoint is False else 1)

    def __len__(self) -> int:
        return self._npoints

    @property
    def shape(self):
        return (self._sig.shape[0], self._npoints, self.channels)

    def _norm(self, start, end):
        n = self._npoints
        start = 0 if start is None else (start + n if start < 0 else start)
        end = n if end is None else (end + n if end < 0 else end)
        return start, end

    def signatures(self, starts, ends) -> torch.Tensor:
        """[B, Q, S]: Sig(x[starts[q]:ends[q]]) for every query q."""
        qs, qe = zip(*(self._norm(a, b) for a, b in zip(starts, ends))) if len(starts) else ((), ())
        return _PathQuery.apply(self._sig, self._inv, self.channels, self.depth, tuple(qs), tuple(qe))

    def signature(self, start=None, end=None) -> torch.Tensor:
        """[B, S]: Sig(x[start:end])."""
        return self.signatures([start], [end])[:, 0]

    def logsignature(self, start=None, end=None, mode: str = "words") -> torch.Tensor:
        return signature_to_logsignature(self.signature(start, end), self.channels, self.depth, mode)

    def update(self, new_points: torch.Tensor) -> None:
        """Append points [B, L', C]: extends both prefix tensors from their last rows."""
        last = self._last
        ns = signature(new_points, self.depth, stream=True, basepoint=last, initial=self._sig[:, -1])
        ni = signature(new_points, self.depth, stream=True, basepoint=last, inverse=True, initial=self._inv[:, -1])
        self._sig = torch.cat([self._sig, ns], dim=1)
        self._inv = torch.cat([self._inv, ni], dim=1)
        self._last = new_points[:, -1, :]
        self._npoints += new_points.shape[1]
