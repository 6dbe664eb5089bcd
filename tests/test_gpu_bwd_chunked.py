"""GPU parity of the time-parallel reversible backward: chunk
signatures, their ordered prefix / suffix products, the gradient at every chunk end, all chunks
reversed at once, shared boundary points fixed up.  Against the float64 oracle's plain reverse
mode (which stores every prefix and shares nothing with the reversible scheme)."""
import numpy as np
import pytest
import torch

import oracle
from synth import brownian_paths, normal
from tests.parity import BWD_TOL, path_rel_err

pytestmark = pytest.mark.gpu
sb = pytest.importorskip("paper_2001_00706_b200")


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


@pytest.mark.parametrize("C,N,B,L", [(3, 4, 2, 700), (8, 3, 1, 300), (2, 5, 4, 257), (4, 4, 3, 1000)])
def test_small_batch_chunked_backward(C, N, B, L):
    """B < 148 paths: the backward splits time into chunks to fill the SMs."""
    x = brownian_paths(B, L, C, seed=C + L)
    S = sb.sig_signature_channels(C, N)
    g = normal((B, S), 5)
    xt = _cuda(x).requires_grad_(True)
    sb.signature(xt, N).backward(_cuda(g))
    ref, _ = oracle.signature_vjp(g, x, N, threads=8)
    err = path_rel_err(xt.grad.cpu().numpy(), ref)
    print(f"PARITY chunked bwd C={C} N={N} B={B} L={L}: {err:.3e}")
    assert err < BWD_TOL


def test_long_path_chunked():
    """One long path (40000 points): split into time chunks for parallelism."""
    C, N, B, L = 3, 4, 1, 40000
    x = brownian_paths(B, L, C, seed=9)
    S = sb.sig_signature_channels(C, N)
    g = normal((B, S), 10)
    xt = _cuda(x).requires_grad_(True)
    sb.signature(xt, N).backward(_cuda(g))
    ref, _ = oracle.signature_vjp(g, x, N)
    assert path_rel_err(xt.grad.cpu().numpy(), ref) < BWD_TOL


@pytest.mark.parametrize("inverse", [False, True])
def test_chunked_backward_with_options(inverse):
    """Chunks with a given basepoint, an initial signature and the inverse option."""
    C, N, B, L = 3, 4, 2, 400
    x = brownian_paths(B, L, C, seed=11)
    bp = (normal((B, C), 12) * 0.3).astype(np.float32)
    ini = oracle.signature(brownian_paths(B, 6, C, seed=13), N).astype(np.float32)
    S = sb.sig_signature_channels(C, N)
    g = normal((B, S), 14)
    xt = _cuda(x).requires_grad_(True)
    bt = _cuda(bp).requires_grad_(True)
    it = _cuda(ini).requires_grad_(True)
    sb.signature(xt, N, basepoint=bt, inverse=inverse, initial=it).backward(_cuda(g))
    rx, rb, ri = oracle.signature_vjp_ex(g, x, N, basepoint=bp, inverse=inverse, initial=ini)
    err = max(path_rel_err(xt.grad.cpu().numpy(), rx), path_rel_err(bt.grad.cpu().numpy()[:, None], rb[:, None]),
              path_rel_err(it.grad.cpu().numpy()[:, None], ri[:, None]))
    assert err < BWD_TOL


def test_chunked_backward_is_deterministic():
    C, N, B, L = 4, 4, 2, 900
    x = _cuda(brownian_paths(B, L, C, seed=15))
    S = sb.sig_signature_channels(C, N)
    g = _cuda(normal((B, S), 16))
    out = sb.sig_signature(x, N)
    a, _ = sb.sig_signature_backward(g, x, out, N)
    b, _ = sb.sig_signature_backward(g, x, out, N)
    assert torch.equal(a, b)


def test_long_path_unchunked_plain_call():
    """The plain C call sig_signature_backward (no workspace, so no time chunks) on a path far
    longer than one CTA could stage whole: K2 stages its increments tile by tile (K2)."""
    C, N, B, L = 3, 4, 2, 40000
    x = brownian_paths(B, L, C, seed=19)
    S = sb.sig_signature_channels(C, N)
    g = normal((B, S), 20)
    xt = _cuda(x)
    gt = _cuda(g)
    out = sb.sig_signature(xt, N)
    gp = torch.empty_like(xt)
    Lib = sb.lib()
    st = Lib.sig_signature_backward(sb._ptr(gt), sb._ptr(xt), sb._ptr(out), B, L, C, N, 0, sb.BP_NONE, None,
                                    sb._ptr(gp), None, sb._stream(xt.device))
    assert st == 0, Lib.sig_last_error()
    torch.cuda.synchronize()
    ref, _ = oracle.signature_vjp(g, x, N)
    err = path_rel_err(gp.cpu().numpy(), ref)
    print(f"PARITY unchunked long-path bwd: {err:.3e}")
    assert err < BWD_TOL
