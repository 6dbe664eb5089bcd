"""Float64 CPU oracle for the Signatory hot path (arXiv 2001.00706) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package.  The product package ``paper_2001_00706_b200``
never imports it, and it shares no code with the CUDA path.

The arithmetic lives in ``oracle.c`` (plain C, float64, compiled ``-O2`` without fast-math) and in
``lyndon.py`` (pure-Python brute force for the Lyndon tables).  This module is marshalling only:
it upcasts the caller's (float32) inputs to float64, prepends basepoints (reading R4),
and loops over the batch -- optionally on a thread pool, since ctypes releases the GIL.

Every function follows the paper's definitions, cited as P:Lnnn = line of PAPER.md:
  signature           P:L68-75, P:L98-101 (eq-computation), conventional exp-then-[x]
  signature_vjp       plain reverse mode through the above (not reversibility)
  log / log_vjp       truncated series log(1+x) (reading R7)
  logsignature        log, then words = psi, brackets = solve phi(x) = log,
                      expand = log itself
  combine             [x]; multi_combine = left fold
  signature_ex        inverse (Sig(x)^-1 = Sig(reversed x), per prefix when streaming)
                      and initial (initial [x] Sig; with inverse Sig^-1 [x] initial,
                      reading R18); signature_vjp_ex = plain reverse mode through it
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import lyndon as _lyndon

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")

_dp = ctypes.POINTER(ctypes.c_double)


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so with gcc (plain -O2, no fast-math)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-o", _SO, _SRC, "-lm"])
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        L.orc_sig_channels.restype = ctypes.c_int64
        L.orc_sig_channels.argtypes = [ctypes.c_int, ctypes.c_int]
        L.orc_level_offset.restype = ctypes.c_int64
        L.orc_level_offset.argtypes = [ctypes.c_int, ctypes.c_int]
        L.orc_tensor_exp.argtypes = [_dp, ctypes.c_int, ctypes.c_int, _dp]
        L.orc_tensor_exp_vjp.argtypes = [_dp, _dp, ctypes.c_int, ctypes.c_int, _dp]
        L.orc_mul.argtypes = [_dp, _dp, ctypes.c_int, ctypes.c_int, _dp]
        L.orc_mul_vjp.argtypes = [_dp, _dp, _dp, ctypes.c_int, ctypes.c_int, _dp, _dp]
        L.orc_signature.restype = ctypes.c_int
        L.orc_signature.argtypes = [_dp, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp]
        L.orc_signature_vjp.restype = ctypes.c_int
        L.orc_signature_vjp.argtypes = [_dp, _dp, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                        ctypes.c_int, _dp]
        L.orc_log.argtypes = [_dp, ctypes.c_int, ctypes.c_int, _dp]
        L.orc_log_vjp.argtypes = [_dp, _dp, ctypes.c_int, ctypes.c_int, _dp]
        L.orc_fused_cost.restype = ctypes.c_int64
        L.orc_fused_cost.argtypes = [ctypes.c_int64, ctypes.c_int]
        L.orc_conventional_cost.restype = ctypes.c_int64
        L.orc_conventional_cost.argtypes = [ctypes.c_int64, ctypes.c_int]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_dp)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


# ------------------------------------------------------------------------------------------------
# sizes and single-element algebra
# ------------------------------------------------------------------------------------------------
def sig_channels(C: int, N: int) -> int:
    return int(lib().orc_sig_channels(C, N))


def level_offset(C: int, k: int) -> int:
    return int(lib().orc_level_offset(C, k))


def levels(x: np.ndarray, C: int, N: int):
    """Split the last axis of a flat truncated tensor into its N levels (views)."""
    return [x[..., level_offset(C, k):level_offset(C, k) + C ** k] for k in range(1, N + 1)]


def tensor_exp(z, N: int) -> np.ndarray:
    z = _f64(z)
    C = z.shape[-1]
    out = np.empty(sig_channels(C, N))
    lib().orc_tensor_exp(_p(z), C, N, _p(out))
    return out


def tensor_exp_vjp(g, z, N: int) -> np.ndarray:
    g, z = _f64(g), _f64(z)
    gz = np.zeros(z.shape[-1])
    lib().orc_tensor_exp_vjp(_p(g), _p(z), z.shape[-1], N, _p(gz))
    return gz


def mul(a, b, C: int, N: int) -> np.ndarray:
    """a [x] b for group elements (implicit scalar 1)."""
    a, b = _f64(a), _f64(b)
    out = np.empty(sig_channels(C, N))
    lib().orc_mul(_p(a), _p(b), C, N, _p(out))
    return out


def mul_vjp(g, a, b, C: int, N: int):
    g, a, b = _f64(g), _f64(a), _f64(b)
    ga = np.zeros_like(a)
    gb = np.zeros_like(b)
    lib().orc_mul_vjp(_p(g), _p(a), _p(b), C, N, _p(ga), _p(gb))
    return ga, gb


def log(a, C: int, N: int) -> np.ndarray:
    a = _f64(a)
    out = np.empty_like(a)
    lib().orc_log(_p(a), C, N, _p(out))
    return out


def log_vjp(g, a, C: int, N: int) -> np.ndarray:
    g, a = _f64(g), _f64(a)
    ga = np.empty_like(a)
    lib().orc_log_vjp(_p(g), _p(a), C, N, _p(ga))
    return ga


def fused_cost(d: int, N: int) -> int:
    return int(lib().orc_fused_cost(d, N))


def conventional_cost(d: int, N: int) -> int:
    return int(lib().orc_conventional_cost(d, N))


# ------------------------------------------------------------------------------------------------
# batched transforms
# ------------------------------------------------------------------------------------------------
def _with_basepoint(path: np.ndarray, basepoint):
    """Reading R4: basepoint=None -> as is; True/'zero' -> prepend the origin; array [B,C] ->
    prepend that point.  Returns float64 [B, L', C]."""
    path = _f64(path)
    if basepoint is None or basepoint is False:
        return path
    B, _, C = path.shape
    if basepoint is True or (isinstance(basepoint, str) and basepoint == "zero"):
        bp = np.zeros((B, 1, C))
    else:
        bp = _f64(basepoint).reshape(B, 1, C)
    return np.ascontiguousarray(np.concatenate([bp, path], axis=1))


def _map(fn, n: int, threads: int):
    if threads <= 1 or n <= 1:
        return [fn(i) for i in range(n)]
    with ThreadPoolExecutor(max_workers=threads) as ex:
        return list(ex.map(fn, range(n)))


def signature(path, depth: int, stream: bool = False, basepoint=None, threads: int = 1) -> np.ndarray:
    """Sig^N of each stream in path[B, L, C] (float64 result).  [B, S] or, with stream=True,
    [B, L'-1, S] where L' counts the basepoint if one is given."""
    x = _with_basepoint(path, basepoint)
    B, L, C = x.shape
    if L < 2:
        raise ValueError("stream needs at least two points (P:L69); add a basepoint")
    S = sig_channels(C, depth)
    out = np.empty((B, L - 1, S) if stream else (B, S))

    def one(b):
        o = np.empty((L - 1, S) if stream else S)
        rc = lib().orc_signature(_p(np.ascontiguousarray(x[b])), L, C, depth, int(stream), _p(o))
        assert rc == 0
        out[b] = o

    _map(one, B, threads)
    return out


def signature_vjp(grad_out, path, depth: int, stream: bool = False, basepoint=None, threads: int = 1):
    """Returns (grad_path [B,L,C], grad_basepoint [B,C] or None) for loss = <grad_out, Sig>."""
    x = _with_basepoint(path, basepoint)
    B, L, C = x.shape
    g = _f64(grad_out)
    gx = np.empty((B, L, C))

    def one(b):
        o = np.empty((L, C))
        rc = lib().orc_signature_vjp(_p(np.ascontiguousarray(g[b])), _p(np.ascontiguousarray(x[b])),
                                     L, C, depth, int(stream), _p(o))
        assert rc == 0
        gx[b] = o

    _map(one, B, threads)
    if basepoint is None or basepoint is False:
        return gx, None
    gbp = gx[:, 0, :].copy()
    return np.ascontiguousarray(gx[:, 1:, :]), (None if basepoint is True or isinstance(basepoint, str) else gbp)


def signature_ex(path, depth: int, stream: bool = False, basepoint=None, inverse: bool = False,
                 initial=None, threads: int = 1) -> np.ndarray:
    """signature with the inverse / initial options (reading R18).

    inverse: Sig(x)^{-1} = Sig(x reversed), computed by definition on the reversed
    (augmented) stream -- for stream=True on every reversed prefix (x_{t+1}, ..., x_0).
    initial [B, S]: the result is initial [x] Sig (the update case); with inverse the
    result is Sig^{-1} [x] initial (initial being the inverse of the earlier signature, since
    (A [x] B)^{-1} = B^{-1} [x] A^{-1})."""
    x = _with_basepoint(path, basepoint)
    B, L, C = x.shape
    if not inverse:
        base = signature(x, depth, stream=stream, threads=threads)
    elif not stream:
        base = signature(np.ascontiguousarray(x[:, ::-1]), depth, threads=threads)
    else:
        base = np.stack([signature(np.ascontiguousarray(x[:, t + 1::-1]), depth, threads=threads)
                         for t in range(L - 1)], axis=1)
    if initial is None:
        return base
    ini = _f64(initial)
    out = np.empty_like(base)
    for b in range(B):
        rows = base[b] if stream else base[b][None]
        res = [mul(r, ini[b], C, depth) if inverse else mul(ini[b], r, C, depth) for r in rows]
        out[b] = np.stack(res) if stream else res[0]
    return out


def signature_vjp_ex(grad_out, path, depth: int, stream: bool = False, basepoint=None, inverse: bool = False,
                     initial=None, threads: int = 1):
    """Reverse mode through signature_ex: (grad_path, grad_basepoint or None, grad_initial or None)."""
    x = _with_basepoint(path, basepoint)
    B, L, C = x.shape
    g = _f64(grad_out)
    ginit = None
    if initial is not None:
        # through the [x] with initial: gradient w.r.t. the plain (inverse) signature and initial
        ini = _f64(initial)
        base = signature_ex(path, depth, stream=stream, basepoint=basepoint, inverse=inverse, threads=threads)
        gbase = np.empty_like(base)
        ginit = np.zeros_like(ini)
        for b in range(B):
            rows = range(L - 1) if stream else [None]
            for t in rows:
                r = base[b, t] if stream else base[b]
                gr = g[b, t] if stream else g[b]
                if inverse:
                    ga, gi = mul_vjp(gr, r, ini[b], C, depth)
                else:
                    gi, ga = mul_vjp(gr, ini[b], r, C, depth)
                ginit[b] += gi
                if stream:
                    gbase[b, t] = ga
                else:
                    gbase[b] = ga
        g = gbase
    if not inverse:
        gx, _ = signature_vjp(g, x, depth, stream=stream, threads=threads)
    elif not stream:
        gr, _ = signature_vjp(g, np.ascontiguousarray(x[:, ::-1]), depth, threads=threads)
        gx = gr[:, ::-1]
    else:
        gx = np.zeros((B, L, C))
        for t in range(L - 1):
            gr, _ = signature_vjp(g[:, t], np.ascontiguousarray(x[:, t + 1::-1]), depth, threads=threads)
            gx[:, :t + 2] += gr[:, ::-1]
    gx = np.ascontiguousarray(gx)
    if basepoint is None or basepoint is False:
        return gx, None, ginit
    gbp = None if (basepoint is True or isinstance(basepoint, str)) else gx[:, 0, :].copy()
    return np.ascontiguousarray(gx[:, 1:, :]), gbp, ginit


def combine(a, b, C: int, N: int) -> np.ndarray:
    """Batched signature_combine: a [x] b row by row."""
    a, b = _f64(a), _f64(b)
    return np.stack([mul(a[i], b[i], C, N) for i in range(a.shape[0])])


def multi_combine(sigs, C: int, N: int) -> np.ndarray:
    """multi_signature_combine: left fold sigs[0] [x] sigs[1] [x] ... over axis 0."""
    sigs = _f64(sigs)
    acc = sigs[0].copy()
    for j in range(1, sigs.shape[0]):
        acc = combine(acc, sigs[j], C, N)
    return acc


# ------------------------------------------------------------------------------------------------
# logsignature (Appendix A.2)
# ------------------------------------------------------------------------------------------------
def logsignature(path, depth: int, mode: str = "words", stream: bool = False, basepoint=None,
                 threads: int = 1) -> np.ndarray:
    sig = signature(path, depth, stream=stream, basepoint=basepoint, threads=threads)
    C = np.asarray(path).shape[-1]
    return logsignature_from_signature(sig, C, depth, mode)


def logsignature_from_signature(sig, C: int, depth: int, mode: str) -> np.ndarray:
    sig = _f64(sig)
    flat = sig.reshape(-1, sig.shape[-1])
    lg = np.stack([log(r, C, depth) for r in flat])
    if mode == "expand":
        out = lg
    elif mode == "words":
        out = _lyndon.psi(lg, C, depth)
    elif mode == "brackets":
        out = _lyndon.brackets_solve(lg, C, depth)
    else:
        raise ValueError(mode)
    return out.reshape(sig.shape[:-1] + (out.shape[-1],))


def logsignature_vjp(grad_out, path, depth: int, mode: str = "words", stream: bool = False,
                     basepoint=None, threads: int = 1):
    """Reverse mode through logsignature: projection adjoint, then log VJP, then signature VJP."""
    C = np.asarray(path).shape[-1]
    sig = signature(path, depth, stream=stream, basepoint=basepoint, threads=threads)
    g = _f64(grad_out)
    gflat = g.reshape(-1, g.shape[-1])
    if mode == "expand":
        glog = gflat
    elif mode == "words":
        glog = _lyndon.psi_adjoint(gflat, C, depth)
    elif mode == "brackets":
        glog = _lyndon.brackets_solve_adjoint(gflat, C, depth)
    else:
        raise ValueError(mode)
    sflat = sig.reshape(-1, sig.shape[-1])
    gsig = np.stack([log_vjp(glog[i], sflat[i], C, depth) for i in range(sflat.shape[0])])
    gsig = gsig.reshape(sig.shape)
    return signature_vjp(gsig, path, depth, stream=stream, basepoint=basepoint, threads=threads)
