"""Pins for the oracle's signature and group product (CPU only).

Each test checks the oracle against something other than itself: the paper's closed forms and
worked examples (tests/golden/), textbook identities (Levy area), invariants the paper states
(Chen, reversal, reparametrisation), and a brute-force evaluation of the iterated-integral
definition that does not use Chen's identity (tests/bruteforce.py).
"""
import math
import os

import numpy as np
import pytest

import oracle
from synth import brownian_paths, uniform_paths
from tests.bruteforce import iterated_integrals, levy_area, rel_err

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _rand_path(L, C, seed, scale=1.0):
    return np.random.default_rng(seed).standard_normal((L, C)) * scale


# ---------------------------------------------------------------- closed forms / worked examples
def test_exp_closed_form_golden():
    """Sig((x1,x2)) = exp(x2-x1), P:L89-96 (tests/golden/exp_closed_form.txt)."""
    rows = [l for l in open(os.path.join(GOLDEN, "exp_closed_form.txt")) if l.strip() and l[0] != "#"]
    assert len(rows) == 2
    for row in rows:
        head, x1, x2, exp = [p.split() for p in row.split("|")]
        C, N = int(head[0]), int(head[1])
        path = np.array([[float(v) for v in x1], [float(v) for v in x2]])
        got = oracle.signature(path[None], N)[0]
        np.testing.assert_allclose(got, [float(v) for v in exp], rtol=0, atol=1e-15)


def test_exp_scalar_channel_is_scalar_exponential():
    """C = 1: levels are D^k/k!, the terms of the scalar exponential series."""
    for D in (-1.7, 0.3, 2.5):
        got = oracle.signature(np.array([[[0.0], [D]]]), 8)[0]
        np.testing.assert_allclose(got, [D ** k / math.factorial(k) for k in range(1, 9)], rtol=1e-14)


def test_level_one_is_total_increment():
    """Sig_1 = x_L - x_1 (k = 1 of eq-signaturedef)."""
    x = brownian_paths(3, 17, 4, seed=11)
    s = oracle.signature(x, 3)
    np.testing.assert_allclose(s[:, :4], (x[:, -1] - x[:, 0]).astype(np.float64), rtol=1e-12, atol=1e-14)


def test_level_two_levy_area_and_symmetric_part():
    """Antisymmetric part of level 2 = Levy area; symmetric part = 1/2 S1 (x) S1 (textbook)."""
    for C, L, seed in [(2, 9, 1), (3, 12, 2), (5, 6, 3)]:
        x = _rand_path(L, C, seed)
        s = oracle.signature(x[None], 2)[0]
        S1 = s[:C]
        S2 = s[C:].reshape(C, C)
        np.testing.assert_allclose(0.5 * (S2 - S2.T), levy_area(x), atol=1e-13)
        np.testing.assert_allclose(0.5 * (S2 + S2.T), 0.5 * np.outer(S1, S1), atol=1e-13)


@pytest.mark.parametrize("C,N,L", [(1, 5, 4), (2, 4, 5), (3, 4, 6), (2, 5, 7), (4, 3, 5)])
def test_bruteforce_iterated_integrals(C, N, L):
    """Oracle (exp-then-[x]) equals the iterated-integral definition evaluated by brute force."""
    x = _rand_path(L, C, seed=100 * C + N)
    np.testing.assert_allclose(oracle.signature(x[None], N)[0], iterated_integrals(x, N),
                               rtol=1e-12, atol=1e-13)


def test_straight_line_collinear():
    """Collinear points (0, v, 2v, 3v): increments commute, Sig = exp(3v)."""
    v = np.array([0.3, -0.7, 1.1])
    x = np.stack([0 * v, v, 2 * v, 3 * v])
    np.testing.assert_allclose(oracle.signature(x[None], 5)[0], oracle.tensor_exp(3 * v, 5), rtol=1e-12)


# ---------------------------------------------------------------- group structure
def test_mul_worked_example_d2_n2():
    """exp(e1) [x] exp(e2), d=2, N=2: word 12 = 1, word 21 = 0, diagonal 1/2 (expand eq-tensorproduct
    by hand: level 2 = e1e1/2 + e1 (x) e2 + e2e2/2)."""
    e1, e2 = np.array([1.0, 0.0]), np.array([0.0, 1.0])
    out = oracle.mul(oracle.tensor_exp(e1, 2), oracle.tensor_exp(e2, 2), 2, 2)
    np.testing.assert_allclose(out, [1, 1, 0.5, 1, 0, 0.5], atol=0)


def test_mul_identity_commuting_associative():
    rng = np.random.default_rng(5)
    C, N = 3, 4
    S = oracle.sig_channels(C, N)
    A, B, D = (rng.standard_normal(S) for _ in range(3))
    zero = np.zeros(S)
    np.testing.assert_allclose(oracle.mul(A, zero, C, N), A, atol=0)
    np.testing.assert_allclose(oracle.mul(zero, A, C, N), A, atol=0)
    lhs = oracle.mul(oracle.mul(A, B, C, N), D, C, N)
    rhs = oracle.mul(A, oracle.mul(B, D, C, N), C, N)
    assert rel_err(lhs, rhs) < 1e-12
    # d = 1 commutes: exp(a) [x] exp(b) = exp(a + b)
    a, b = np.array([0.7]), np.array([-1.9])
    np.testing.assert_allclose(oracle.mul(oracle.tensor_exp(a, 6), oracle.tensor_exp(b, 6), 1, 6),
                               oracle.tensor_exp(a + b, 6), rtol=1e-13, atol=1e-15)
    # non-commutative for d = 2
    e1, e2 = np.array([1.0, 0.0]), np.array([0.0, 1.0])
    assert not np.allclose(oracle.mul(oracle.tensor_exp(e1, 2), oracle.tensor_exp(e2, 2), 2, 2),
                           oracle.mul(oracle.tensor_exp(e2, 2), oracle.tensor_exp(e1, 2), 2, 2))


@pytest.mark.parametrize("C,N,L", [(2, 3, 8), (3, 4, 10), (4, 5, 9), (1, 4, 6)])
def test_chen_identity_every_split(C, N, L):
    """Sig(x_1..x_L) = Sig(x_1..x_j) [x] Sig(x_j..x_L) for every j (eq-grouplike)."""
    x = _rand_path(L, C, seed=C * 7 + N)
    full = oracle.signature(x[None], N)[0]
    for j in range(2, L):  # 1-based j in {2..L-1}
        left = oracle.signature(x[None, :j], N)[0]
        right = oracle.signature(x[None, j - 1:], N)[0]
        assert rel_err(oracle.mul(left, right, C, N), full) < 1e-12


def test_reversal_is_inverse():
    """Sig(x) [x] Sig(reversed x) = 1."""
    for C, N in [(2, 4), (3, 5), (5, 3)]:
        x = _rand_path(9, C, seed=C + N)
        s = oracle.signature(x[None], N)[0]
        r = oracle.signature(x[None, ::-1].copy(), N)[0]
        assert np.max(np.abs(oracle.mul(s, r, C, N))) < 1e-12
        assert np.max(np.abs(oracle.mul(r, s, C, N))) < 1e-12


def test_reparametrisation_and_translation_invariance():
    """Inserting a segment midpoint, duplicating a point, or translating leaves Sig unchanged
    (P:L75 invariance to the choice of time points)."""
    C, N = 3, 5
    x = _rand_path(7, C, seed=42)
    s = oracle.signature(x[None], N)[0]
    mid = np.insert(x, 3, 0.5 * (x[2] + x[3]), axis=0)
    dup = np.insert(x, 4, x[4], axis=0)
    assert rel_err(oracle.signature(mid[None], N)[0], s) < 1e-12
    assert rel_err(oracle.signature(dup[None], N)[0], s) < 1e-12
    assert rel_err(oracle.signature((x + np.array([3.0, -1.0, 0.25]))[None], N)[0], s) < 1e-12


def test_stream_mode_rows_are_prefix_signatures():
    """stream=True returns Sig(x_1,x_2), ..., Sig(x_1..x_L)."""
    x = uniform_paths(2, 7, 3, seed=9)
    st = oracle.signature(x, 4, stream=True)
    assert st.shape == (2, 6, oracle.sig_channels(3, 4))
    for j in range(2, 8):
        np.testing.assert_allclose(st[:, j - 2], oracle.signature(x[:, :j], 4), rtol=1e-14, atol=0)


def test_basepoint_prepends_point():
    """basepoint (reading R4): zero prepends the origin, a given point prepends that point."""
    x = brownian_paths(2, 5, 3, seed=3)
    bp = np.array([[0.1, 0.2, -0.3], [1.0, 0.0, 0.5]], dtype=np.float32)
    got0 = oracle.signature(x, 3, basepoint=True)
    ref0 = oracle.signature(np.concatenate([np.zeros((2, 1, 3), np.float32), x], axis=1), 3)
    np.testing.assert_array_equal(got0, ref0)
    got1 = oracle.signature(x, 3, basepoint=bp)
    ref1 = oracle.signature(np.concatenate([bp[:, None, :], x], axis=1), 3)
    np.testing.assert_array_equal(got1, ref1)
    # a single point with a basepoint is legal: Sig = exp(x_0 - bp)
    one = oracle.signature(x[:, :1], 3, basepoint=bp)
    np.testing.assert_allclose(one[0], oracle.tensor_exp(x[0, 0].astype(np.float64) - bp[0], 3), rtol=1e-15)


def test_multi_combine_three_way_split():
    C, N = 3, 4
    x = _rand_path(13, C, seed=8)
    parts = [x[0:5], x[4:9], x[8:13]]
    sigs = np.stack([oracle.signature(p[None], N) for p in parts])  # [3, 1, S]
    np.testing.assert_allclose(oracle.multi_combine(sigs, C, N)[0], oracle.signature(x[None], N)[0],
                               rtol=1e-12, atol=1e-14)
