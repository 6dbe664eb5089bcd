"""Pins for the oracle's inverse / initial options (reading R18).

Each pin is a property the paper states, checked with independent primitives: the group inverse
(Sig(x) [x] Sig(x)^{-1} = identity), Chen's identity for the update case, and central finite
differences for the reverse mode."""
import numpy as np
import pytest

import oracle
from synth import brownian_paths, normal
from tests.bruteforce import finite_difference


def _identity_err(a):
    return np.abs(a).max()  # the identity has every level k >= 1 zero


@pytest.mark.parametrize("C,N", [(2, 4), (3, 3)])
def test_inverse_is_group_inverse(C, N):
    x = brownian_paths(3, 7, C, seed=11)
    sig = oracle.signature(x, N)
    inv = oracle.signature_ex(x, N, inverse=True)
    for b in range(3):
        assert _identity_err(oracle.mul(sig[b], inv[b], C, N)) < 1e-12
        assert _identity_err(oracle.mul(inv[b], sig[b], C, N)) < 1e-12


def test_stream_inverse_is_prefix_inverse():
    C, N = 2, 3
    x = brownian_paths(2, 6, C, seed=12)
    sigs = oracle.signature(x, N, stream=True)
    invs = oracle.signature_ex(x, N, stream=True, inverse=True)
    for b in range(2):
        for t in range(5):
            assert _identity_err(oracle.mul(sigs[b, t], invs[b, t], C, N)) < 1e-12


@pytest.mark.parametrize("stream", [False, True])
def test_initial_is_chen_update(stream):
    """Sig(x_1..x_L) from Sig(x_1..x_j) and the new points x_j..x_L."""
    C, N, j = 3, 3, 4
    x = brownian_paths(2, 9, C, seed=13)
    old = oracle.signature(x[:, :j + 1], N)
    new = oracle.signature_ex(x[:, j:], N, stream=stream, initial=old)
    full = oracle.signature(x, N, stream=stream)
    ref = full[:, j:] if stream else full
    assert np.abs(new - ref).max() < 1e-12


def test_inverse_with_initial_updates_the_inverse():
    C, N, j = 2, 4, 3
    x = brownian_paths(2, 8, C, seed=14)
    old_inv = oracle.signature_ex(x[:, :j + 1], N, inverse=True)
    new = oracle.signature_ex(x[:, j:], N, inverse=True, initial=old_inv)
    ref = oracle.signature_ex(x, N, inverse=True)
    assert np.abs(new - ref).max() < 1e-12


@pytest.mark.parametrize("stream,inverse,bp", [(False, True, None), (True, True, "given"), (False, False, "given"),
                                               (True, False, None)])
def test_vjp_ex_finite_differences(stream, inverse, bp):
    C, N, B, L = 2, 3, 2, 4
    x = brownian_paths(B, L, C, seed=15)
    basepoint = normal((B, C), 16) * 0.3 if bp == "given" else None
    ini = oracle.signature(brownian_paths(B, 3, C, seed=17), N)
    S = oracle.sig_channels(C, N)
    g = normal((B, L - 1 + (bp is not None), S) if stream else (B, S), 18)

    def loss(xx, bpp, ii):
        return float((oracle.signature_ex(xx, N, stream=stream, basepoint=bpp, inverse=inverse, initial=ii) * g).sum())

    gx, gb, gi = oracle.signature_vjp_ex(g, x, N, stream=stream, basepoint=basepoint, inverse=inverse, initial=ini)
    fx = finite_difference(lambda v: loss(v, basepoint, ini), x)
    assert np.abs(gx - fx).max() < 1e-6 * max(1.0, np.abs(fx).max())
    fi = finite_difference(lambda v: loss(x, basepoint, v), ini)
    assert np.abs(gi - fi).max() < 1e-6 * max(1.0, np.abs(fi).max())
    if basepoint is not None:
        fb = finite_difference(lambda v: loss(x, v, ini), basepoint)
        assert np.abs(gb - fb).max() < 1e-6 * max(1.0, np.abs(fb).max())
