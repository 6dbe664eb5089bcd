"""Pins for the oracle's tensor log, Lyndon tables, projections and brackets solve (CPU only)."""
import itertools
import os

import numpy as np
import pytest

import oracle
from oracle import lyndon
from tests.bruteforce import finite_difference, rel_err

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _rand(shape, seed, scale=1.0):
    return np.random.default_rng(seed).standard_normal(shape) * scale


def _lie_exp(y, C, N):
    """exp of a zero-scalar element y: sum_{n=0}^N y^n / n!, products via np.multiply.outer
    level by level (used only to check log against its inverse)."""
    lv = lambda t, k: t[oracle.level_offset(C, k):oracle.level_offset(C, k) + C ** k]

    def prod(a, b):
        out = np.zeros_like(a)
        for k in range(1, N + 1):
            acc = np.zeros(C ** k)
            for i in range(1, k):
                acc += np.multiply.outer(lv(a, i), lv(b, k - i)).reshape(-1)
            out[oracle.level_offset(C, k):oracle.level_offset(C, k) + C ** k] = acc
        return out

    out = y.copy()
    p = y.copy()
    fact = 1.0
    for n in range(2, N + 1):
        p = prod(p, y)
        fact *= n
        out += p / fact
    return out


# ---------------------------------------------------------------- log
def test_log_of_single_segment_is_increment():
    """log(exp z) = (z, 0, ..., 0): a single segment's logsignature is its increment."""
    for C, N in [(2, 5), (3, 4), (4, 3)]:
        z = _rand(C, C + N)
        lg = oracle.log(oracle.tensor_exp(z, N), C, N)
        np.testing.assert_allclose(lg[:C], z, rtol=1e-14)
        assert np.max(np.abs(lg[C:])) < 1e-13


def test_log_identity_is_zero():
    assert np.all(oracle.log(np.zeros(oracle.sig_channels(3, 4)), 3, 4) == 0)


def test_log_bch_closed_form():
    """Baker-Campbell-Hausdorff (textbook): log(exp z [x] exp w) = z + w + 1/2 [z,w]
    + 1/12 ([z,[z,w]] + [w,[w,z]]) + (level >= 4 terms).  Reading R8 (SPEC's level-2 statement
    describes the signature, not its log)."""
    C, N = 3, 4
    z, w = _rand(C, 1), _rand(C, 2)
    lg = oracle.log(oracle.mul(oracle.tensor_exp(z, N), oracle.tensor_exp(w, N), C, N), C, N)
    br = lambda a, b: np.multiply.outer(a, b) - np.multiply.outer(b, a)
    zw = br(z, w)
    np.testing.assert_allclose(lg[:C], z + w, rtol=1e-14)
    np.testing.assert_allclose(lg[C:C + C * C], 0.5 * zw.reshape(-1), atol=1e-14)
    l3 = (np.multiply.outer(z, br(z, w)) - np.multiply.outer(br(z, w), z)
          + np.multiply.outer(w, br(w, z)) - np.multiply.outer(br(w, z), w)) / 12.0
    off3 = oracle.level_offset(C, 3)
    np.testing.assert_allclose(lg[off3:off3 + C ** 3], l3.reshape(-1), atol=1e-14)


def test_exp_of_log_roundtrip():
    """log is the inverse of the (series) exponential on group-like elements (P:L117 footnote)."""
    C, N = 3, 5
    x = _rand((1, 8, C), 5, 0.6)
    s = oracle.signature(x, N)[0]
    np.testing.assert_allclose(_lie_exp(oracle.log(s, C, N), C, N), s, rtol=1e-12, atol=1e-13)


def test_worked_logsig_d2_n2():
    """Stream ((0,0),(1,0),(1,1)), d=2, N=2: expanded level 2 = +-1/2 at words 12/21, brackets [12] =
    1/2 (equals 1/2 [e1, e2] by BCH)."""
    x = np.array([[[0.0, 0.0], [1.0, 0.0], [1.0, 1.0]]])
    ex = oracle.logsignature(x, 2, mode="expand")[0]
    np.testing.assert_allclose(ex, [1, 1, 0, 0.5, -0.5, 0], atol=1e-15)
    np.testing.assert_allclose(oracle.logsignature(x, 2, mode="brackets")[0], [1, 1, 0.5], atol=1e-15)
    np.testing.assert_allclose(oracle.logsignature(x, 2, mode="words")[0], [1, 1, 0.5], atol=1e-15)


@pytest.mark.parametrize("mode", ["words", "brackets", "expand"])
def test_single_segment_logsig_modes(mode):
    """L=2: (Delta_1..Delta_d, 0, ..., 0) in (length, lex) Lyndon order."""
    x = np.array([[[0.0, 0.0], [0.7, -1.3]]])
    out = oracle.logsignature(x, 3, mode=mode)[0]
    n = 5 if mode != "expand" else 14
    assert out.shape == (n,)
    np.testing.assert_allclose(out[:2], [0.7, -1.3], rtol=1e-14)
    assert np.max(np.abs(out[2:])) < 1e-15


def test_log_vjp_finite_differences():
    C, N = 3, 4
    S = oracle.sig_channels(C, N)
    A = oracle.signature(_rand((1, 5, C), 1, 0.5), N)[0]
    g = _rand(S, 2)
    ga = oracle.log_vjp(g, A, C, N)
    fd = finite_difference(lambda a: float(g @ oracle.log(a, C, N)), A)
    assert rel_err(ga, fd) < 1e-6


@pytest.mark.parametrize("mode", ["words", "brackets", "expand"])
@pytest.mark.parametrize("C,N,L", [(2, 4, 5), (3, 3, 6)])
def test_logsignature_vjp_finite_differences(mode, C, N, L):
    x = _rand((1, L, C), seed=C + 5 * N, scale=0.6)
    w = oracle.logsignature(x, N, mode=mode).shape[-1]
    g = _rand((1, w), 77)
    gx, _ = oracle.logsignature_vjp(g, x, N, mode=mode)
    fd = finite_difference(lambda y: float(np.sum(g * oracle.logsignature(y, N, mode=mode))), x)
    assert rel_err(gx, fd) < 1e-5


# ---------------------------------------------------------------- Lyndon words and brackets
def test_lyndon_paper_examples_golden():
    for line in open(os.path.join(GOLDEN, "lyndon_paper_examples.txt")):
        line = line.strip()
        if not line or line[0] == "#":
            continue
        kind, rest = line.split(":", 1)
        if kind == "order":
            ws = [tuple(int(c) - 1 for c in p.split()) for p in rest.split("<")]
            assert all(a < b for a, b in zip(ws, ws[1:]))
        else:
            w = tuple(int(c) - 1 for c in rest.split())
            assert lyndon.is_lyndon(w) == (kind == "lyndon")


def test_lyndon_count_is_witt():
    """Number of Lyndon words of length <= N = w(d, N) (Witt's formula)."""
    for C in range(1, 5):
        for N in range(1, 7):
            assert len(lyndon.lyndon_words(C, N)) == lyndon.witt(C, N)


def test_lyndon_small_lists():
    assert lyndon.lyndon_words(2, 3) == ((0,), (1,), (0, 1), (0, 0, 1), (0, 1, 1))  # w(2,3)=5
    assert len(lyndon.lyndon_words(3, 2)) == 6
    assert lyndon.lyndon_words(1, 5) == ((0,),)
    # SURVEY 8 table values of Witt's formula used for output sizes
    assert lyndon.witt(4, 7) == 3304 and lyndon.witt(8, 5) == 7764 and lyndon.witt(3, 6) == 196
    assert lyndon.witt(4, 4) == 90 and lyndon.witt(6, 4) == 406


def test_standard_factorisation_examples():
    assert lyndon.factor((0, 0, 1)) == ((0,), (0, 1))
    assert lyndon.factor((0, 1, 1)) == ((0, 1), (1,))
    assert lyndon.factor((0, 1)) == ((0,), (1,))
    # both factors are Lyndon for every Lyndon word ("It is a fact")
    for w in lyndon.lyndon_words(3, 5):
        if len(w) > 1:
            a, b = lyndon.factor(w)
            assert lyndon.is_lyndon(a) and lyndon.is_lyndon(b) and a + b == w


def test_phi_worked_example_golden():
    lines = [l.strip() for l in open(os.path.join(GOLDEN, "phi_a1a2a2.txt")) if l.strip() and l[0] != "#"]
    w = tuple(int(c) - 1 for c in lines[0].split(":")[1].split())
    expect = {}
    for l in lines[1:]:
        word, coef = l.split(":")
        expect[tuple(int(c) - 1 for c in word.split())] = int(coef)
    assert lyndon.phi(w) == expect


def test_triangularity_and_homogeneity():
    """psi o phi is unit lower-triangular in lex order; phi(w) is homogeneous."""
    for C in (2, 3):
        for N in range(1, 6):
            for w in lyndon.lyndon_words(C, N):
                p = lyndon.phi(w)
                assert all(len(u) == len(w) for u in p)
                assert p.get(w) == 1
                for u in p:
                    if lyndon.is_lyndon(u):
                        assert u >= w  # zero coefficient on Lyndon words earlier than w
            for _, M in lyndon.psi_phi_blocks(C, N):
                assert np.allclose(M, np.tril(M)) and np.all(np.diag(M) == 1)


@pytest.mark.parametrize("C,N", [(2, 4), (3, 3), (2, 5), (3, 4)])
def test_brackets_reconstruct_full_log(C, N):
    """sum_l alpha_l phi(l) = log Sig on EVERY coordinate (image(log) = image(phi)),
    agrees with a least-squares solve of the tall system, and words = M . brackets."""
    x = _rand((3, 6, C), seed=C * N, scale=0.8)
    lg = oracle.logsignature(x, N, mode="expand")
    al = oracle.logsignature(x, N, mode="brackets")
    wd = oracle.logsignature(x, N, mode="words")
    assert rel_err(lyndon.phi_expand_flat(al, C, N), lg) < 1e-12
    # least squares on the tall system phi(x) = log, built column by column
    words = lyndon.lyndon_words(C, N)
    Phi = np.stack([lyndon.phi_expand_flat(np.eye(len(words))[j], C, N) for j in range(len(words))], axis=1)
    ls = np.linalg.lstsq(Phi, lg.T, rcond=None)[0].T
    assert rel_err(ls, al) < 1e-10
    col = 0
    for wk, M in lyndon.psi_phi_blocks(C, N):
        n = len(wk)
        np.testing.assert_allclose(wd[:, col:col + n], al[:, col:col + n] @ M.T, atol=1e-12)
        col += n
