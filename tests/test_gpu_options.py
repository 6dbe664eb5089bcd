"""GPU parity of the inverse / initial signature options (R18)
against the float64 oracle (oracle.signature_ex / signature_vjp_ex), forward and backward."""
import numpy as np
import pytest
import torch

import oracle
from synth import brownian_paths, normal
from tests.parity import BWD_TOL, FWD_TOL, level_rel_err, path_rel_err

pytestmark = pytest.mark.gpu
sb = pytest.importorskip("paper_2001_00706_b200")


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def _initial(B, C, N, seed):
    # a genuine signature (group-like), as in the update use case
    return oracle.signature(brownian_paths(B, 5, C, seed=seed), N).astype(np.float32)


CASES = [  # C, N, B, L
    (2, 4, 3, 12),
    (4, 4, 4, 20),
    (8, 3, 2, 10),
    (3, 5, 2, 9),
]
OPTS = [  # stream, inverse, with_initial, basepoint
    (False, True, False, None),
    (False, True, True, "given"),
    (False, False, True, None),
    (True, True, False, None),
    (True, True, True, "zero"),
    (True, False, True, "given"),
]


def _bp(kind, B, C):
    if kind is None:
        return None, None
    if kind == "zero":
        return True, True
    v = normal((B, C), 77) * 0.5
    return _cuda(v), v.astype(np.float32)


@pytest.mark.parametrize("stream,inverse,with_initial,bpk", OPTS)
@pytest.mark.parametrize("C,N,B,L", CASES)
def test_options_forward(C, N, B, L, stream, inverse, with_initial, bpk):
    x = brownian_paths(B, L, C, seed=C * 7 + N)
    ini = _initial(B, C, N, 5) if with_initial else None
    bpt, bpn = _bp(bpk, B, C)
    got = sb.sig_signature(_cuda(x), N, stream=stream, basepoint=bpt, inverse=inverse,
                           initial=None if ini is None else _cuda(ini)).cpu().numpy()
    ref = oracle.signature_ex(x, N, stream=stream, basepoint=bpn, inverse=inverse, initial=ini)
    err = level_rel_err(got.reshape(-1, got.shape[-1]), ref.reshape(-1, ref.shape[-1]), C, N)
    print(f"PARITY options fwd C={C} N={N} stream={stream} inverse={inverse} initial={with_initial}: {err:.3e}")
    assert err < FWD_TOL


@pytest.mark.parametrize("stream,inverse,with_initial,bpk", OPTS)
@pytest.mark.parametrize("C,N,B,L", CASES)
def test_options_backward(C, N, B, L, stream, inverse, with_initial, bpk):
    x = brownian_paths(B, L, C, seed=C * 7 + N + 1)
    ini = _initial(B, C, N, 6) if with_initial else None
    bpt, bpn = _bp(bpk, B, C)
    S = sb.sig_signature_channels(C, N)
    M = L - 1 + (bpk is not None)
    g = normal((B, M, S) if stream else (B, S), 88)
    xt = _cuda(x).requires_grad_(True)
    it = None if ini is None else _cuda(ini).requires_grad_(True)
    if bpk == "given":
        bpt = bpt.clone().requires_grad_(True)
    out = sb.signature(xt, N, stream=stream, basepoint=bpt, inverse=inverse, initial=it)
    out.backward(_cuda(g))
    rx, rb, ri = oracle.signature_vjp_ex(g, x, N, stream=stream, basepoint=bpn, inverse=inverse, initial=ini)
    err = path_rel_err(xt.grad.cpu().numpy(), rx)
    if ini is not None:
        err = max(err, path_rel_err(it.grad.cpu().numpy()[:, None, :], ri[:, None, :]))
    if bpk == "given":
        err = max(err, path_rel_err(bpt.grad.cpu().numpy()[:, None, :], rb[:, None, :]))
    print(f"PARITY options bwd C={C} N={N} stream={stream} inverse={inverse} initial={with_initial}: {err:.3e}")
    assert err < BWD_TOL


@pytest.mark.parametrize("inverse", [False, True])
def test_options_time_chunked_plan(inverse):
    """A batch too small to fill the GPU is split into time chunks and folded: the initial
    state goes to each path's first chunk; the inverse runs through the same fold."""
    C, N, B, L = 3, 4, 2, 700
    x = brownian_paths(B, L, C, seed=99)
    ini = _initial(B, C, N, 7)
    got = sb.sig_signature(_cuda(x), N, inverse=inverse, initial=_cuda(ini)).cpu().numpy()
    ref = oracle.signature_ex(x, N, inverse=inverse, initial=ini)
    assert level_rel_err(got, ref, C, N) < FWD_TOL


def test_update_matches_full_signature():
    """The update use case end to end on the GPU: old signature + new points == full signature."""
    C, N, B, L, j = 4, 4, 3, 40, 25
    x = brownian_paths(B, L, C, seed=100)
    xt = _cuda(x)
    old = sb.sig_signature(xt[:, :j + 1], N)
    new = sb.sig_signature(xt[:, j:], N, initial=old)
    full = sb.sig_signature(xt, N)
    assert level_rel_err(new.cpu().numpy(), full.cpu().numpy(), C, N) < FWD_TOL
    inv_old = sb.sig_signature(xt[:, :j + 1], N, inverse=True)
    inv_new = sb.sig_signature(xt[:, j:], N, inverse=True, initial=inv_old)
    inv_full = sb.sig_signature(xt, N, inverse=True)
    assert level_rel_err(inv_new.cpu().numpy(), inv_full.cpu().numpy(), C, N) < FWD_TOL
