"""GPU parity of Path (O(1) interval queries from prefix signatures and prefix
inverse signatures) and of signature_to_logsignature.

The oracle side computes each interval's signature directly from the sub-stream (by definition),
so the group-like identity InvertSig(x_0..x_s) [x] Sig(x_0..x_{e-1}) = Sig(x_s..x_{e-1}) that the
GPU path relies on is checked, not assumed."""
import numpy as np
import pytest
import torch

import oracle
from synth import brownian_paths, normal
from tests.parity import BWD_TOL, FWD_TOL, block_rel_err, level_rel_err, path_rel_err

pytestmark = pytest.mark.gpu
sb = pytest.importorskip("paper_2001_00706_b200")


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def _query_err(got, x, s, e, C, N):
    """Per level k: |gpu - Sig(x[s:e])| / max(|Sig_k|, T_k, floor), T_k = max_i |Inv_i| |Sig'_{k-i}| the
    largest term of the [x] sum InvertSig(x[:s+1]) [x] Sig(x[:e]).  The query inherits that sum's
    cancellation (the paper's caution; reading R19), so the bar is relative to
    it; for s = 0 the query is a stored prefix row and T_k = |Sig_k|."""
    ref = oracle.signature(x[:, s:e], N)
    sig_e = oracle.signature(x[:, :e], N)
    inv_s = oracle.signature_ex(x[:, :s + 1], N, inverse=True) if s > 0 else np.zeros_like(sig_e)
    off = np.cumsum([0] + [C ** k for k in range(1, N + 1)])
    nrm = lambda a, k: np.abs(a[:, off[k - 1]:off[k]]).max(axis=1) if k > 0 else np.ones(a.shape[0])
    worst = 0.0
    floor = 1e-4 * max(nrm(ref, k).max() for k in range(1, N + 1))
    for k in range(1, N + 1):
        T = np.max([nrm(inv_s, i) * nrm(sig_e, k - i) for i in range(0, k + 1)], axis=0)
        den = np.maximum(np.maximum(nrm(ref, k), T), floor)
        num = np.abs(got[:, off[k - 1]:off[k]] - ref[:, off[k - 1]:off[k]]).max(axis=1)
        worst = max(worst, float((num / den).max()))
    return worst


def _intervals(n, rng, k):
    out = [(0, n), (0, 2), (n - 2, n), (1, n - 1)]
    while len(out) < k:
        s = int(rng.integers(0, n - 1))
        e = int(rng.integers(s + 2, n + 1))
        out.append((s, e))
    return out


@pytest.mark.parametrize("C,N,B,L", [(2, 4, 3, 30), (4, 4, 2, 25), (3, 3, 2, 40)])
def test_path_queries(C, N, B, L):
    x = brownian_paths(B, L, C, seed=50 + C)
    p = sb.Path(_cuda(x), N)
    iv = _intervals(L, np.random.default_rng(C), 24)
    got = p.signatures([a for a, _ in iv], [b for _, b in iv]).cpu().numpy()
    for q, (s, e) in enumerate(iv):
        assert _query_err(got[:, q], x, s, e, C, N) < FWD_TOL, (s, e)
    one = p.signature(3, 17).cpu().numpy()
    assert _query_err(one, x, 3, 17, C, N) < FWD_TOL


def test_path_with_basepoint_and_negative_indices():
    C, N, B, L = 3, 4, 2, 20
    x = brownian_paths(B, L, C, seed=61)
    bp = normal((B, C), 62).astype(np.float32)
    p = sb.Path(_cuda(x), N, basepoint=_cuda(bp))
    xa = np.concatenate([bp[:, None, :], x], axis=1)
    assert len(p) == L + 1
    got = p.signature(None, -3).cpu().numpy()
    assert level_rel_err(got, oracle.signature(xa[:, :L + 1 - 3], N), C, N) < FWD_TOL


def test_path_logsignature():
    C, N, B, L = 4, 4, 2, 30
    x = brownian_paths(B, L, C, seed=63)
    p = sb.Path(_cuda(x), N)
    for mode in ("words", "brackets", "expand"):
        got = p.logsignature(5, 21, mode).cpu().numpy()
        ref = oracle.logsignature(x[:, 5:21], N, mode=mode)
        lv = [len(w) for w in oracle.lyndon.lyndon_words(C, N)] if mode != "expand" else None
        if mode == "expand":
            err = level_rel_err(got, ref, C, N)
        else:
            blocks = [(lv.index(k), len(lv) - lv[::-1].index(k)) for k in range(1, N + 1)]
            err = block_rel_err(got, ref, blocks)
        assert err < FWD_TOL, mode


def test_path_update():
    """Path(x[:j]) updated with x[j:] answers every query like Path(x)."""
    C, N, B, L, j = 3, 4, 2, 36, 20
    x = brownian_paths(B, L, C, seed=64)
    full = sb.Path(_cuda(x), N)
    part = sb.Path(_cuda(x[:, :j]), N)
    part.update(_cuda(x[:, j:]))
    assert len(part) == L
    iv = _intervals(L, np.random.default_rng(7), 16) + [(3, j + 5), (j - 1, L)]
    a = full.signatures([s for s, _ in iv], [e for _, e in iv]).cpu().numpy()
    b = part.signatures([s for s, _ in iv], [e for _, e in iv]).cpu().numpy()
    for q, (s, e) in enumerate(iv):
        assert _query_err(b[:, q], x, s, e, C, N) < FWD_TOL, (s, e)
        assert _query_err(a[:, q], x, s, e, C, N) < FWD_TOL, (s, e)


@pytest.mark.parametrize("C,N", [(2, 4), (4, 3)])
def test_path_query_backward(C, N):
    """d/dx of sum_q <g_q, Sig(x[s_q:e_q])>: through the query [x]-VJP, then the reversible
    backward of both prefix scans (plain and inverse) -- against the sum of sub-stream VJPs."""
    B, L = 2, 18
    x = brownian_paths(B, L, C, seed=65 + C)
    iv = [(0, L), (2, 9), (2, 14), (5, 9), (0, 6), (11, 18), (5, 9)]  # repeated rows and a duplicate query
    S = oracle.sig_channels(C, N)
    g = normal((B, len(iv), S), 66)
    xt = _cuda(x).requires_grad_(True)
    p = sb.Path(xt, N)
    out = p.signatures([s for s, _ in iv], [e for _, e in iv])
    out.backward(_cuda(g))
    ref = np.zeros_like(x, dtype=np.float64)
    for q, (s, e) in enumerate(iv):
        gx, _ = oracle.signature_vjp(g[:, q], x[:, s:e], N)
        ref[:, s:e] += gx
    assert path_rel_err(xt.grad.cpu().numpy(), ref) < BWD_TOL


def test_path_query_validation():
    x = _cuda(brownian_paths(1, 10, 2, seed=1))
    p = sb.Path(x, 3)
    with pytest.raises(sb.SigError):
        p.signature(4, 5)  # a single point
    with pytest.raises(sb.SigError):
        p.signature(0, 11)  # past the end


@pytest.mark.parametrize("mode", ["words", "brackets", "expand"])
def test_signature_to_logsignature(mode):
    C, N, B, L = 3, 4, 3, 15
    x = brownian_paths(B, L, C, seed=70)
    w = sb.sig_logsignature_channels(C, N, mode)
    g = normal((B, w), 71)
    xt = _cuda(x).requires_grad_(True)
    ls = sb.signature_to_logsignature(sb.signature(xt, N), C, N, mode)
    ref = oracle.logsignature(x, N, mode=mode)
    assert np.abs(ls.detach().cpu().numpy() - ref).max() < FWD_TOL * max(1.0, np.abs(ref).max())
    ls.backward(_cuda(g))
    rg, _ = oracle.logsignature_vjp(g, x, N, mode=mode)
    assert path_rel_err(xt.grad.cpu().numpy(), rg) < BWD_TOL
