"""GPU parity for the logsignature (K4/K5) and the combine kernels (K3) against the oracle."""
import numpy as np
import pytest
import torch

import oracle
from oracle import lyndon
from synth import brownian_paths, normal
from tests.parity import BWD_TOL, FWD_TOL, block_rel_err, level_rel_err, path_rel_err

pytestmark = pytest.mark.gpu
sb = pytest.importorskip("paper_2001_00706_b200")


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _blocks(C, N, mode):
    if mode == "expand":
        out, off = [], 0
        for k in range(1, N + 1):
            out.append((off, off + C ** k))
            off += C ** k
        return out
    lv = [len(w) for w in lyndon.lyndon_words(C, N)]
    return [(lv.index(k), len(lv) - lv[::-1].index(k)) for k in range(1, N + 1) if k in lv]


# (3,7), (5,5), (6,4) have ownership prefix P < N in the owned-prefix backward (non power-of-two C)
LOG_CASES = [(4, 7, 4, 64), (3, 4, 5, 30), (2, 5, 6, 20), (8, 3, 3, 40), (4, 4, 8, 128), (3, 7, 3, 20), (5, 5, 3, 16),
             (6, 4, 3, 16), (8, 5, 3, 40)]


@pytest.mark.parametrize("mode", ["words", "brackets", "expand"])
@pytest.mark.parametrize("C,N,B,L", LOG_CASES)
def test_logsignature_forward(mode, C, N, B, L):
    x = brownian_paths(B, L, C, seed=C + N)
    got = sb.sig_logsignature(_cuda(x), N, mode).cpu().numpy()
    ref = oracle.logsignature(x, N, mode=mode, threads=8)
    assert got.shape == ref.shape
    err = block_rel_err(got, ref, _blocks(C, N, mode))
    print(f"PARITY logsig fwd {mode} C={C} N={N} B={B} L={L}: {err:.3e}")
    assert err < FWD_TOL


@pytest.mark.parametrize("mode", ["words", "brackets", "expand"])
@pytest.mark.parametrize("C,N,B,L", [(4, 7, 3, 48), (3, 4, 4, 20), (2, 5, 3, 15), (8, 3, 2, 30), (3, 7, 2, 12),
                                     (5, 5, 2, 10), (8, 5, 2, 6)])
def test_logsignature_backward(mode, C, N, B, L):
    """K5 in its three forms: compiled per (C, N) for power-of-two C (4,7), (2,5), (8,3); the runtime
    owned-prefix kernel (3,4), (3,7), (5,5); the general fallback (8,5) (owned layout too large)."""
    x = brownian_paths(B, L, C, seed=3 * C + N)
    w = sb.sig_logsignature_channels(C, N, mode)
    g = normal((B, w), seed=104)
    xt = _cuda(x).requires_grad_(True)
    out = sb.logsignature(xt, N, mode)
    out.backward(_cuda(g))
    ref, _ = oracle.logsignature_vjp(g, x, N, mode=mode, threads=8)
    err = path_rel_err(xt.grad.cpu().numpy(), ref)
    print(f"PARITY logsig bwd {mode} C={C} N={N} B={B} L={L}: {err:.3e}")
    assert err < BWD_TOL


def test_logsignature_one_channel_exact_zeros():
    """C = 1: the logsignature is (x_L - x_1, 0, ..., 0) exactly (one channel commutes); the zero
    levels are checked absolutely against the scale of the signature level they come from."""
    x = brownian_paths(2, 9, 1, seed=3)
    for mode in ("words", "brackets", "expand"):
        got = sb.sig_logsignature(_cuda(x), 3, mode).cpu().numpy()
        d = (x[:, -1, 0] - x[:, 0, 0]).astype(np.float64)
        np.testing.assert_allclose(got[:, 0], d, rtol=1e-5, atol=1e-6)
        if got.shape[1] > 1:
            assert np.max(np.abs(got[:, 1:])) < 1e-5 * max(1.0, float(np.max(np.abs(d))) ** 3)


def test_logsignature_stream_and_single_segment():
    C, N, B, L = 3, 4, 2, 12
    x = brownian_paths(B, L, C, seed=9)
    got = sb.sig_logsignature(_cuda(x), N, "words", stream=True).cpu().numpy()
    ref = oracle.logsignature(x, N, mode="words", stream=True)
    assert block_rel_err(got, ref, _blocks(C, N, "words")) < FWD_TOL
    seg = np.array([[[0.0, 0.0], [0.7, -1.3]]], dtype=np.float32)
    out = sb.sig_logsignature(_cuda(seg), 3, "brackets").cpu().numpy()[0]
    np.testing.assert_allclose(out[:2], [0.7, -1.3], rtol=1e-6)
    assert np.max(np.abs(out[2:])) < 1e-6


def test_c4_full_size_sampled():
    """BASELINE config c4 (B=512, L=256, C=4, N=7, words) full batch fwd+bwd, every 32nd path checked."""
    C, N, B, L = 4, 7, 512, 256
    x = brownian_paths(B, L, C, seed=4)
    g = normal((B, 3304), seed=104)
    xt = _cuda(x).requires_grad_(True)
    out = sb.logsignature(xt, N, "words")
    out.backward(_cuda(g))
    idx = np.arange(0, B, 32)
    ref = oracle.logsignature(x[idx], N, mode="words", threads=16)
    ef = block_rel_err(out.detach().cpu().numpy()[idx], ref, _blocks(C, N, "words"))
    rg, _ = oracle.logsignature_vjp(g[idx], x[idx], N, mode="words", threads=16)
    eb = path_rel_err(xt.grad.cpu().numpy()[idx], rg)
    print(f"PARITY c4 full-size sampled: fwd {ef:.3e} bwd {eb:.3e}")
    assert ef < FWD_TOL and eb < BWD_TOL


@pytest.mark.parametrize("C,N,B", [(3, 4, 5), (8, 5, 2), (2, 7, 3), (4, 1, 4)])
def test_combine_and_backward(C, N, B):
    S = sum(C ** k for k in range(1, N + 1))
    xa = brownian_paths(B, 9, C, seed=1)
    xb = brownian_paths(B, 7, C, seed=2)
    a = oracle.signature(xa, N).astype(np.float32)
    b = oracle.signature(xb, N).astype(np.float32)
    got = sb.sig_signature_combine(_cuda(a), _cuda(b), C, N).cpu().numpy()
    ref = oracle.combine(a, b, C, N)
    assert level_rel_err(got, ref, C, N) < FWD_TOL
    g = normal((B, S), seed=3)
    ga, gb = sb.sig_signature_combine_backward(_cuda(g), _cuda(a), _cuda(b), C, N)
    ra = np.stack([oracle.mul_vjp(g[i], a[i], b[i], C, N)[0] for i in range(B)])
    rb = np.stack([oracle.mul_vjp(g[i], a[i], b[i], C, N)[1] for i in range(B)])
    assert path_rel_err(ga.cpu().numpy(), ra) < BWD_TOL
    assert path_rel_err(gb.cpu().numpy(), rb) < BWD_TOL


@pytest.mark.parametrize("n", [1, 2, 5, 40, 129])
def test_multi_combine_chen(n):
    """Folding the signatures of consecutive pieces equals the signature of the whole (Chen)."""
    C, N, B = 3, 4, 3
    pieces = n
    L = 4 * pieces + 1
    x = brownian_paths(B, L, C, seed=n)
    sigs = np.stack([oracle.signature(x[:, 4 * j:4 * j + 5], N) for j in range(pieces)]).astype(np.float32)
    got = sb.multi_signature_combine(_cuda(sigs), C, N).cpu().numpy()
    assert level_rel_err(got, oracle.signature(x, N), C, N) < FWD_TOL


_POW2_INSTANCES = [(C, N) for C in (1, 2, 4, 8) for N in range(1, 13) if sum(C ** k for k in range(1, N + 1)) <= 6000]


@pytest.mark.parametrize("C,N", _POW2_INSTANCES)
def test_logsignature_backward_every_compiled_instance(C, N):
    """Every compiled (C, N) instance of the owned-prefix K5 (expand and words), small paths."""
    x = brownian_paths(2, 6, C, seed=C * 31 + N)
    for mode in ("expand", "words"):
        w = sb.sig_logsignature_channels(C, N, mode)
        g = normal((2, w), seed=7)
        xt = _cuda(x).requires_grad_(True)
        sb.logsignature(xt, N, mode).backward(_cuda(g))
        ref, _ = oracle.logsignature_vjp(g, x, N, mode=mode)
        got = xt.grad.cpu().numpy()
        if C == 1:
            # one channel: log = (increment, 0, ..., 0), so the path gradient is +-g_1 at the end
            # points, reached through cancelling O(|g|) terms; scale the error by |g| (not the
            # possibly tiny |g_1| of one path)
            err = np.abs(got - ref).max() / max(np.abs(ref).max(), np.abs(g).max())
        else:
            err = path_rel_err(got, ref)
        assert err < BWD_TOL, (C, N, mode, err)


@pytest.mark.parametrize("mode", ["words", "brackets", "expand"])
@pytest.mark.parametrize("C,N,B,L,bp", [(3, 4, 2, 12, None), (4, 3, 3, 9, "zero"), (2, 5, 2, 10, "given")])
def test_logsignature_stream_backward(mode, C, N, B, L, bp):
    """Stream-mode logsignature (every prefix) forward and backward."""
    x = brownian_paths(B, L, C, seed=40 + C)
    bpn = None if bp is None else (True if bp == "zero" else normal((B, C), 41).astype(np.float32))
    bpt = bpn if not isinstance(bpn, np.ndarray) else _cuda(bpn)
    w = sb.sig_logsignature_channels(C, N, mode)
    M = L - 1 + (bp is not None)
    g = normal((B, M, w), seed=42)
    xt = _cuda(x).requires_grad_(True)
    out = sb.logsignature(xt, N, mode, stream=True, basepoint=bpt)
    got = out.detach().cpu().numpy().reshape(-1, w)
    # K4 takes the float32 signature rows: against the oracle's log of its own signature rounded
    # to float32 the bar is 1e-4; against the exact log, short prefixes amplify that rounding
    # (reading R20), hence 5e-4 end to end
    sig32 = oracle.signature(x, N, stream=True, basepoint=bpn).astype(np.float32)
    ref32 = oracle.logsignature_from_signature(sig32.reshape(-1, sig32.shape[-1]), C, N, mode)
    assert block_rel_err(got, ref32, _blocks(C, N, mode)) < FWD_TOL
    ref = oracle.logsignature(x, N, mode=mode, stream=True, basepoint=bpn)
    assert block_rel_err(got, ref.reshape(-1, w), _blocks(C, N, mode)) < 5 * FWD_TOL
    out.backward(_cuda(g))
    rg, _ = oracle.logsignature_vjp(g, x, N, mode=mode, stream=True, basepoint=bpn)
    assert path_rel_err(xt.grad.cpu().numpy(), rg) < BWD_TOL


@pytest.mark.parametrize("stream", [False, True])
def test_logsignature_inverse(stream):
    """log(Sig^-1): for group-like Sig it is -log(Sig) (expand basis)."""
    C, N, B, L = 3, 4, 2, 11
    x = brownian_paths(B, L, C, seed=43)
    inv = sb.logsignature(_cuda(x), N, "expand", stream=stream, inverse=True).cpu().numpy()
    ref = -oracle.logsignature(x, N, mode="expand", stream=stream)
    S = ref.shape[-1]
    assert level_rel_err(inv.reshape(-1, S), ref.reshape(-1, S), C, N) < FWD_TOL


@pytest.mark.parametrize("C,N,n", [(8, 4, 7), (8, 5, 3), (2, 9, 17)])
def test_multi_combine_fold_paths(C, N, n):
    """The compiled group fold (S small enough for groups in shared memory: (8,4), (2,9)) and the
    pairwise fold in global memory (S = 37448 at (8,5)) against the oracle's left fold."""
    B = 2
    sigs = np.stack([oracle.signature(brownian_paths(B, 6, C, seed=100 + j), N) for j in range(n)]).astype(np.float32)
    got = sb.multi_signature_combine(_cuda(sigs), C, N).cpu().numpy()
    ref = oracle.multi_combine(sigs, C, N)
    assert level_rel_err(got, ref, C, N) < FWD_TOL


@pytest.mark.parametrize("mode", ["words", "brackets", "expand"])
@pytest.mark.parametrize("C,N,B,L", [(6, 4, 3, 600), (3, 5, 2, 700), (4, 4, 2, 800), (8, 3, 4, 400)])
def test_logsignature_stream_many_rows(mode, C, N, B, L):
    """Stream-mode logsignature with more than 8 x 148 rows: K4 runs one warp per row
    (logsig_rows.cuh).  Against the oracle's log of its own signature rounded to float32 (R20)."""
    x = brownian_paths(B, L, C, seed=60 + C)
    w = sb.sig_logsignature_channels(C, N, mode)
    assert B * (L - 1) >= 8 * 148
    got = sb.logsignature(_cuda(x), N, mode, stream=True).cpu().numpy().reshape(-1, w)
    sig32 = oracle.signature(x, N, stream=True).astype(np.float32).reshape(-1, sb.sig_signature_channels(C, N))
    rows = np.r_[0:64, sig32.shape[0] - 64:sig32.shape[0], 500:sig32.shape[0]:97]  # sampled rows, both ends
    ref32 = oracle.logsignature_from_signature(sig32[rows], C, N, mode)
    err = block_rel_err(got[rows], ref32, _blocks(C, N, mode))
    print(f"PARITY stream logsig many rows C={C} N={N} {mode}: {err:.3e}")
    assert err < FWD_TOL


def test_logsignature_rows_kernel_matches_per_row_kernel():
    """The warp-per-row K4 and the CTA-per-row K4 compute the same log of the same rows (the row
    count alone selects the kernel): bitwise equality is not required (summation order is the
    same, float64), but agreement to float32 rounding."""
    C, N = 6, 4
    S = sb.sig_signature_channels(C, N)
    sig = oracle.signature(brownian_paths(4, 400, C, seed=70), N, stream=True).astype(np.float32).reshape(-1, S)
    many = sb.sig_logsignature_from_signature(_cuda(sig), C, N, "words").cpu().numpy()
    few = np.concatenate([sb.sig_logsignature_from_signature(_cuda(sig[i:i + 100]), C, N, "words").cpu().numpy()
                          for i in range(0, sig.shape[0], 100)])
    np.testing.assert_allclose(many, few, rtol=2e-6, atol=1e-7)


def test_logsignature_backward_long_path():
    """a logsignature backward on a path longer than one CTA stages whole (L = 40000)
    runs through the chunked/tiled signature backward with the plan's workspace (no SIG_ERR_WORKSPACE)
    and matches the oracle's projection adjoint -> log VJP -> signature VJP."""
    C, N, B, L = 3, 4, 2, 40000
    x = brownian_paths(B, L, C, seed=31)
    w = sb.sig_logsignature_channels(C, N, "words")
    g = normal((B, w), 32)
    xt = _cuda(x)
    out, sig = sb.sig_logsignature(xt, N, "words", return_signature=True)
    gx = sb.sig_logsignature_backward(_cuda(g), xt, sig, N, "words")
    if isinstance(gx, tuple):
        gx = gx[0]
    ref, _ = oracle.logsignature_vjp(g, x, N, mode="words", threads=8)
    err = path_rel_err(gx.cpu().numpy(), ref)
    print(f"PARITY long-path logsig bwd (L={L}): {err:.3e}")
    assert err < BWD_TOL


def test_combine_rows_beyond_grid_y():
    """more rows than gridDim.y allows (65535): the combine kernels grid-stride over rows."""
    C, N, B = 2, 3, 70000
    S = sum(C ** k for k in range(1, N + 1))
    rng = np.random.default_rng(41)
    a = (0.5 * rng.standard_normal((B, S))).astype(np.float32)
    b = (0.5 * rng.standard_normal((B, S))).astype(np.float32)
    got = sb.sig_signature_combine(_cuda(a), _cuda(b), C, N).cpu().numpy()
    idx = np.concatenate([np.arange(8), np.arange(65530, 65545), np.arange(B - 8, B)])
    ref = oracle.combine(a[idx], b[idx], C, N)
    assert level_rel_err(got[idx], ref, C, N) < FWD_TOL
    g = normal((B, S), seed=42)
    ga, gb = sb.sig_signature_combine_backward(_cuda(g), _cuda(a), _cuda(b), C, N)
    ra = np.stack([oracle.mul_vjp(g[i], a[i], b[i], C, N)[0] for i in idx])
    rb = np.stack([oracle.mul_vjp(g[i], a[i], b[i], C, N)[1] for i in idx])
    assert path_rel_err(ga.cpu().numpy()[idx], ra) < BWD_TOL
    assert path_rel_err(gb.cpu().numpy()[idx], rb) < BWD_TOL
