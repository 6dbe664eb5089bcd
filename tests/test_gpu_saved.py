"""GPU parity of the forward with saved chunk states (sig_signature_save) and the backward that
starts from them (sig_signature_backward_saved), include/sig.h: against the oracle, and bit for bit
against the time-parallel backward that recomputes the chunk signatures itself."""
import numpy as np
import pytest
import torch

import oracle
from synth import brownian_paths, normal
from tests.parity import BWD_TOL, FWD_TOL, level_rel_err, path_rel_err

pytestmark = pytest.mark.gpu
sb = pytest.importorskip("paper_2001_00706_b200")


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("C,N,B,L,bp", [(3, 4, 1, 40000, None), (3, 6, 1, 20000, "zero"), (4, 4, 3, 3000, "given"),
                                        (8, 3, 2, 2500, None)])
def test_saved_forward_backward(C, N, B, L, bp):
    x = brownian_paths(B, L, C, seed=51)
    S = sb.sig_signature_channels(C, N)
    g = normal((B, S), 52)
    bpt = None
    if bp == "zero":
        bpa, bpo = True, True
    elif bp == "given":
        bpt = (0.3 * np.random.default_rng(53).standard_normal((B, C))).astype(np.float32)
        bpa, bpo = _cuda(bpt), bpt
    else:
        bpa, bpo = None, None
    xt, gt = _cuda(x), _cuda(g)
    assert sb.lib().sig_signature_saved_bytes(B, L, C, N, {None: 0, "zero": 1, "given": 2}[bp]) > 0  # chunked
    out, saved = sb.sig_signature_save(xt, N, basepoint=bpa)
    assert saved is not None
    ref = oracle.signature(x, N, basepoint=bpo, threads=8)
    ef = level_rel_err(out.cpu().numpy(), ref, C, N)
    gp, gbp = sb.sig_signature_backward_saved(gt, xt, out, saved, N, basepoint=bpa)
    # the recomputing time-parallel backward: same chunking, same kernels, same bits
    gp2, gbp2 = sb.sig_signature_backward(gt, xt, out, N, basepoint=bpa)
    assert torch.equal(gp, gp2)
    if bp == "given":
        assert torch.equal(gbp, gbp2)
    rg, rbp = oracle.signature_vjp(g, x, N, basepoint=bpo, threads=8)
    eb = path_rel_err(gp.cpu().numpy(), rg)
    print(f"PARITY saved C={C} N={N} B={B} L={L} bp={bp}: fwd {ef:.3e} bwd {eb:.3e}")
    assert ef < FWD_TOL and eb < BWD_TOL
    if bp == "given":
        assert path_rel_err(gbp.cpu().numpy(), rbp) < BWD_TOL


def test_saved_not_needed_for_full_batches():
    """A batch that fills the GPU is reversed without chunks: nothing to save, plain calls."""
    C, N, B, L = 2, 3, 2048, 40
    x = brownian_paths(B, L, C, seed=54)
    S = sb.sig_signature_channels(C, N)
    g = normal((B, S), 55)
    xt, gt = _cuda(x), _cuda(g)
    out, saved = sb.sig_signature_save(xt, N)
    assert saved is None
    assert torch.equal(out, sb.sig_signature(xt, N))
    gp, _ = sb.sig_signature_backward_saved(gt, xt, out, None, N)
    gp2, _ = sb.sig_signature_backward(gt, xt, out, N)
    assert torch.equal(gp, gp2)


def test_autograd_uses_saved_chunks():
    """signature(x).backward() keeps the chunk states when a backward will follow: the gradient is
    the time-parallel backward's, bit for bit."""
    C, N, B, L = 3, 5, 1, 30000
    x = brownian_paths(B, L, C, seed=56)
    S = sb.sig_signature_channels(C, N)
    g = normal((B, S), 57)
    xt = _cuda(x).requires_grad_(True)
    out = sb.signature(xt, N)
    L0 = sb.lib().sig_launch_count()
    out.backward(_cuda(g))
    torch.cuda.synchronize()
    n_saved = sb.lib().sig_launch_count() - L0
    ref_out = sb.sig_signature(xt.detach(), N)
    L1 = sb.lib().sig_launch_count()
    gp2, _ = sb.sig_signature_backward(_cuda(g), xt.detach(), out.detach(), N)
    n_recompute = sb.lib().sig_launch_count() - L1
    assert torch.equal(xt.grad, gp2)
    assert n_saved < n_recompute, (n_saved, n_recompute)  # no chunk-signature pass, no prefix scan
    assert level_rel_err(out.detach().cpu().numpy(), ref_out.cpu().numpy(), C, N) < FWD_TOL


def _random_saved_cases(n=8, seed=2026):
    rng = np.random.default_rng(seed)
    shapes = [(2, 6), (2, 9), (3, 4), (3, 6), (4, 4), (4, 5), (5, 3), (6, 3), (7, 3), (8, 3), (8, 4)]
    out = []
    while len(out) < n:
        C, N = shapes[rng.integers(len(shapes))]
        B = int(rng.integers(1, 9))
        L = int(rng.integers(600, 6000))
        bp = [None, "zero", "given"][rng.integers(3)]
        if sb.lib().sig_signature_saved_bytes(B, L, C, N, {None: 0, "zero": 1, "given": 2}[bp]) > 0:
            out.append((C, N, B, L, bp))
    return out


@pytest.mark.parametrize("C,N,B,L,bp", _random_saved_cases())
def test_saved_random_shapes(C, N, B, L, bp):
    """Seeded random small batches of long paths (chunked backward): the saved pair matches the
    recomputing backward bit for bit and the oracle within the bars."""
    x = brownian_paths(B, L, C, seed=C * 100 + N)
    S = sb.sig_signature_channels(C, N)
    g = normal((B, S), C + N)
    bpt = (0.2 * np.random.default_rng(L).standard_normal((B, C))).astype(np.float32) if bp == "given" else None
    bpa = {None: None, "zero": True, "given": None if bpt is None else _cuda(bpt)}[bp]
    bpo = {None: None, "zero": True, "given": bpt}[bp]
    xt, gt = _cuda(x), _cuda(g)
    out, saved = sb.sig_signature_save(xt, N, basepoint=bpa)
    gp, gbp = sb.sig_signature_backward_saved(gt, xt, out, saved, N, basepoint=bpa)
    gp2, gbp2 = sb.sig_signature_backward(gt, xt, out, N, basepoint=bpa)
    assert torch.equal(gp, gp2)
    ref = oracle.signature(x, N, basepoint=bpo, threads=8)
    rg, rbp = oracle.signature_vjp(g, x, N, basepoint=bpo, threads=8)
    assert level_rel_err(out.cpu().numpy(), ref, C, N) < FWD_TOL
    assert path_rel_err(gp.cpu().numpy(), rg) < BWD_TOL
    if bp == "given":
        assert torch.equal(gbp, gbp2)
        assert path_rel_err(gbp.cpu().numpy(), rbp) < BWD_TOL
