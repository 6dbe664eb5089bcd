"""GPU parity over seeded random shapes (C, N, B, L, basepoint, stream): every instantiated (C, N)
family reaches the kernels the library picks for it -- one- and two-prefix scans, grouped and
latency-plan time chunks, the two-prefix / prefix-pair / one-prefix backward, time-chunked
backward for small batches -- and is compared with the float64 oracle (forward at 1e-4 per level,
backward at 5e-4 per path, R9).  Sizes keep the oracle to seconds."""
import numpy as np
import pytest
import torch

import oracle
from synth import brownian_paths, normal
from tests.parity import BWD_TOL, FWD_TOL, level_rel_err, path_rel_err

pytestmark = pytest.mark.gpu
sb = pytest.importorskip("paper_2001_00706_b200")


def _cases(n=24, seed=2026):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        C = int(rng.integers(2, 9))
        N = int(rng.integers(2, 8))
        S = sum(C ** k for k in range(1, N + 1))
        if S > 6000:
            continue
        B = int(rng.choice([1, 3, 7, 33, 150]))
        L = int(rng.choice([2, 5, 17, 64, 200, 700]))
        if B * (L - 1) * S > 4_000_000:  # oracle budget
            continue
        bp = str(rng.choice(["none", "zero", "given"]))
        stream = bool(rng.random() < 0.2) and B * L * S < 2_000_000
        out.append((C, N, B, L, bp, stream))
    return out


@pytest.mark.parametrize("C,N,B,L,bp,stream", _cases())
def test_random_shape_parity(C, N, B, L, bp, stream):
    x = brownian_paths(B, L, C, seed=C * 100 + N * 10 + L)
    S = sb.sig_signature_channels(C, N)
    bpn = None if bp == "none" else (True if bp == "zero" else (normal((B, C), 7) * 0.3).astype(np.float32))
    bpt = bpn if not isinstance(bpn, np.ndarray) else torch.from_numpy(bpn).cuda()
    xt = torch.from_numpy(x).cuda()
    out = sb.sig_signature(xt, N, stream=stream, basepoint=bpt)
    ref = oracle.signature(x, N, stream=stream, basepoint=bpn)
    ef = level_rel_err(out.cpu().numpy().reshape(-1, S), ref.reshape(-1, S), C, N)
    g = normal(tuple(out.shape), 8)
    gp, _ = sb.sig_signature_backward(torch.from_numpy(g).cuda(), xt, out, N, stream=stream, basepoint=bpt)
    rg, _ = oracle.signature_vjp(g, x, N, stream=stream, basepoint=bpn, threads=8)
    eb = path_rel_err(gp.cpu().numpy(), rg)
    print(f"PARITY random C={C} N={N} B={B} L={L} bp={bp} stream={stream}: fwd {ef:.2e} bwd {eb:.2e}")
    assert ef < FWD_TOL and eb < BWD_TOL, (ef, eb)


def _log_cases(n=18, seed=4242):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        C = int(rng.integers(2, 9))
        N = int(rng.integers(2, 7))
        S = sum(C ** k for k in range(1, N + 1))
        if S > 6000:
            continue
        B = int(rng.choice([1, 2, 5, 40]))
        L = int(rng.choice([2, 6, 33, 150]))
        if B * (L - 1) * S > 2_000_000:  # oracle budget
            continue
        mode = str(rng.choice(["words", "brackets", "expand"]))
        stream = bool(rng.random() < 0.3) and B * L * S < 400_000
        bp = str(rng.choice(["none", "zero"]))
        out.append((C, N, B, L, mode, stream, bp))
    return out


@pytest.mark.parametrize("C,N,B,L,mode,stream,bp", _log_cases())
def test_random_shape_logsignature(C, N, B, L, mode, stream, bp):
    """Seeded random shapes through the logsignature (K4 per row / per warp, the three bases) and its
    backward (K5 into the reversible K2), forward and backward against the float64 oracle."""
    x = brownian_paths(B, L, C, seed=C * 1000 + N * 100 + L)
    bpa = True if bp == "zero" else None
    xt = torch.from_numpy(x).cuda().requires_grad_(True)
    out = sb.logsignature(xt, N, mode, stream=stream, basepoint=bpa)
    ref = oracle.logsignature(x, N, mode=mode, stream=stream, basepoint=bpa, threads=8)
    got = out.detach().cpu().numpy()
    w = got.shape[-1]
    den = np.maximum(np.max(np.abs(ref.reshape(-1, w)), axis=1), 1e-30)
    ef = float(np.max(np.max(np.abs(got.reshape(-1, w) - ref.reshape(-1, w)), axis=1) / den))
    g = normal(tuple(out.shape), 9)
    out.backward(torch.from_numpy(g).cuda())
    rg, _ = oracle.logsignature_vjp(g, x, N, mode=mode, stream=stream, basepoint=bpa, threads=8)
    eb = path_rel_err(xt.grad.cpu().numpy(), rg)
    print(f"PARITY random logsig C={C} N={N} B={B} L={L} {mode} stream={stream} bp={bp}: fwd {ef:.2e} bwd {eb:.2e}")
    assert ef < FWD_TOL and eb < BWD_TOL, (ef, eb)
