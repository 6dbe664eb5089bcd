"""Pins for the oracle's VJPs (CPU only): central finite differences of the (already pinned)
forward in float64, the paper-forced special case, linearity, and the top-level invariant."""
import numpy as np
import pytest

import oracle
from tests.bruteforce import finite_difference, rel_err


def _rand(shape, seed, scale=1.0):
    return np.random.default_rng(seed).standard_normal(shape) * scale


def test_special_case_d1_n1_l2():
    """d=1, N=1, L=2: Sig = x2 - x1, so d<1, Sig>/dx = (-1, 1)."""
    gx, _ = oracle.signature_vjp(np.ones((1, 1)), np.array([[[0.3], [1.2]]]), 1)
    np.testing.assert_allclose(gx[0, :, 0], [-1.0, 1.0], atol=0)


@pytest.mark.parametrize("C,N,L,stream", [(2, 3, 5, False), (3, 4, 6, False), (4, 5, 4, False),
                                          (2, 4, 6, True), (3, 3, 5, True), (1, 4, 3, False)])
def test_signature_vjp_finite_differences(C, N, L, stream):
    """Central FD (step 1e-6, float64) of loss = <g, Sig(x)>; max relative error <= 1e-5."""
    x = _rand((1, L, C), seed=C * 10 + N, scale=0.7)
    S = oracle.sig_channels(C, N)
    g = _rand((1, L - 1, S) if stream else (1, S), seed=99)
    gx, _ = oracle.signature_vjp(g, x, N, stream=stream)
    fd = finite_difference(lambda y: float(np.sum(g * oracle.signature(y, N, stream=stream))), x)
    assert rel_err(gx, fd) < 1e-5


def test_signature_vjp_basepoint_given():
    C, N, L = 3, 3, 4
    x = _rand((2, L, C), seed=1, scale=0.5)
    bp = _rand((2, C), seed=2, scale=0.5)
    g = _rand((2, oracle.sig_channels(C, N)), seed=3)
    gx, gbp = oracle.signature_vjp(g, x, N, basepoint=bp)
    fdx = finite_difference(lambda y: float(np.sum(g * oracle.signature(y, N, basepoint=bp))), x)
    fdb = finite_difference(lambda b: float(np.sum(g * oracle.signature(x, N, basepoint=b))), bp)
    assert rel_err(gx, fdx) < 1e-5 and rel_err(gbp, fdb) < 1e-5
    # translation invariance => gradients sum to zero over the (basepoint + path) points
    np.testing.assert_allclose(gx.sum(axis=1) + gbp, 0, atol=1e-12)


def test_signature_vjp_linear_in_grad():
    C, N, L = 3, 4, 6
    x = _rand((1, L, C), seed=4)
    S = oracle.sig_channels(C, N)
    g1, g2 = _rand((1, S), 5), _rand((1, S), 6)
    a, _ = oracle.signature_vjp(2.0 * g1 - 3.0 * g2, x, N)
    b1, _ = oracle.signature_vjp(g1, x, N)
    b2, _ = oracle.signature_vjp(g2, x, N)
    assert rel_err(a, 2.0 * b1 - 3.0 * b2) < 1e-12


def test_gradient_sums_to_zero_translation_invariance():
    """Sig depends only on increments, so the path gradient sums to zero over time."""
    x = _rand((2, 9, 4), seed=7)
    g = _rand((2, oracle.sig_channels(4, 4)), seed=8)
    gx, _ = oracle.signature_vjp(g, x, 4)
    np.testing.assert_allclose(gx.sum(axis=1), 0, atol=1e-11)


def test_mul_and_exp_vjp_finite_differences():
    C, N = 3, 4
    S = oracle.sig_channels(C, N)
    A, B, g = _rand(S, 1), _rand(S, 2), _rand(S, 3)
    ga, gb = oracle.mul_vjp(g, A, B, C, N)
    fa = finite_difference(lambda a: float(g @ oracle.mul(a, B, C, N)), A)
    fb = finite_difference(lambda b: float(g @ oracle.mul(A, b, C, N)), B)
    assert rel_err(ga, fa) < 1e-6 and rel_err(gb, fb) < 1e-6
    z = _rand(C, 4)
    gz = oracle.tensor_exp_vjp(g, z, N)
    fz = finite_difference(lambda v: float(g @ oracle.tensor_exp(v, N)), z)
    assert rel_err(gz, fz) < 1e-6


def test_exp_vjp_zero_increment_identity():
    """z = 0: exp(0) = 1 so d<g, A[x]exp(z)>/dA = g on every level."""
    C, N = 2, 4
    S = oracle.sig_channels(C, N)
    A, g = _rand(S, 11), _rand(S, 12)
    ga, _ = oracle.mul_vjp(g, A, oracle.tensor_exp(np.zeros(C), N), C, N)
    np.testing.assert_allclose(ga, g, atol=0)
