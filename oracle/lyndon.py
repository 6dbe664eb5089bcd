"""Brute-force Lyndon words, brackets phi, projection psi and the Lyndon-basis solve -- ORACLE.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Pure Python on purpose: every step is the
paper's definition, checked by eye, for small alphabets/depths.  Shares nothing with the CUDA
library's host table builder (which uses Duval's algorithm and exact integer inverses).

Letters are 0-based (channel c <-> the paper's a_{c+1}); words are tuples.
  is_lyndon      "a word which comes earlier in lexicographic order than any of its rotations"
                  -- every nontrivial rotation is checked.
  lyndon_words   all Lyndon words of length 1..N ordered by (length, lex)  (reading R5)
  factor         w = w^a w^b with w^b the longest proper Lyndon suffix, found by scanning suffixes
                 from the left (reading R6)
  phi            phi(letter) = letter, phi(w) = [phi(w^a), phi(w^b)], [x, y] = xy - yx
  psi            keep the coefficients of Lyndon words
  brackets_solve the unique x with phi(x) = log Sig, solved per degree through the
                 square system psi(phi(x)) = psi(log Sig), which is unit lower-triangular
                 (P:L563-567); tests check that the full tall system phi(x) = log Sig then holds on
                 every coordinate.
"""
from __future__ import annotations

import functools
import itertools

import numpy as np
from scipy.linalg import solve_triangular


def is_lyndon(w: tuple) -> bool:
    k = len(w)
    return all(w < w[r:] + w[:r] for r in range(1, k))


@functools.lru_cache(maxsize=None)
def lyndon_words(C: int, N: int) -> tuple:
    out = []
    for k in range(1, N + 1):
        for w in itertools.product(range(C), repeat=k):  # lexicographic order
            if is_lyndon(w):
                out.append(w)
    return tuple(out)


def factor(w: tuple):
    """Standard factorisation: smallest j > 1 (1-based) with w_j..w_n Lyndon."""
    assert len(w) >= 2
    for j in range(1, len(w)):
        if is_lyndon(w[j:]):
            return w[:j], w[j:]
    raise AssertionError("unreachable: the last letter is always Lyndon")


def _concat(x: dict, y: dict) -> dict:
    out: dict = {}
    for u, a in x.items():
        for v, b in y.items():
            out[u + v] = out.get(u + v, 0) + a * b
    return out


def commutator(x: dict, y: dict) -> dict:
    out = dict(_concat(x, y))
    for w, c in _concat(y, x).items():
        out[w] = out.get(w, 0) - c
    return {w: c for w, c in out.items() if c != 0}


@functools.lru_cache(maxsize=None)
def _phi_cached(w: tuple):
    if len(w) == 1:
        return ((w, 1),)
    a, b = factor(w)
    return tuple(sorted(commutator(dict(_phi_cached(a)), dict(_phi_cached(b))).items()))


def phi(w: tuple) -> dict:
    """Integer word expansion of the Lyndon bracket of w."""
    return dict(_phi_cached(tuple(w)))


def witt(C: int, N: int) -> int:
    """Witt's formula w(d,N) = sum_k (1/k) sum_{i|k} mu(k/i) d^i."""
    def mobius(n):
        r, p, m = 1, 2, n
        while p * p <= m:
            if m % p == 0:
                m //= p
                if m % p == 0:
                    return 0
                r = -r
            p += 1
        return -r if m > 1 else r

    tot = 0
    for k in range(1, N + 1):
        s = sum(mobius(k // i) * C ** i for i in range(1, k + 1) if k % i == 0)
        assert s % k == 0
        tot += s // k
    return tot


def _flat_index(w: tuple, C: int) -> int:
    """Offset of word w in the level-major flat layout (reading R1)."""
    k = len(w)
    off = sum(C ** j for j in range(1, k))
    idx = 0
    for letter in w:
        idx = idx * C + letter
    return off + idx


@functools.lru_cache(maxsize=None)
def lyndon_flat_indices(C: int, N: int) -> np.ndarray:
    return np.array([_flat_index(w, C) for w in lyndon_words(C, N)], dtype=np.int64)


def psi(x: np.ndarray, C: int, N: int) -> np.ndarray:
    """Gather the Lyndon-word coefficients, in (length, lex) order."""
    return np.asarray(x)[..., lyndon_flat_indices(C, N)]


def psi_adjoint(g: np.ndarray, C: int, N: int) -> np.ndarray:
    g = np.asarray(g, dtype=np.float64)
    S = sum(C ** k for k in range(1, N + 1))
    out = np.zeros(g.shape[:-1] + (S,))
    out[..., lyndon_flat_indices(C, N)] = g
    return out


@functools.lru_cache(maxsize=None)
def psi_phi_blocks(C: int, N: int):
    """Per degree k: (row/col Lyndon words, dense M_k with M_k[r, c] = coefficient of the Lyndon
    word r in phi(c)).  Triangular by P:L563."""
    words = lyndon_words(C, N)
    blocks = []
    for k in range(1, N + 1):
        wk = [w for w in words if len(w) == k]
        pos = {w: i for i, w in enumerate(wk)}
        M = np.zeros((len(wk), len(wk)))
        for j, w in enumerate(wk):
            for u, c in phi(w).items():
                if u in pos:
                    M[pos[u], j] = c
        blocks.append((wk, M))
    return tuple(blocks)


def brackets_solve(logsig: np.ndarray, C: int, N: int) -> np.ndarray:
    """Lyndon-basis coefficients alpha with sum_l alpha_l phi(l) = log Sig."""
    z = psi(logsig, C, N)  # [..., w]
    out = np.empty_like(z)
    col = 0
    for wk, M in psi_phi_blocks(C, N):
        n = len(wk)
        rhs = z[..., col:col + n].reshape(-1, n).T
        sol = solve_triangular(M, rhs, lower=True, unit_diagonal=False)
        out[..., col:col + n] = sol.T.reshape(z.shape[:-1] + (n,))
        col += n
    return out


def brackets_solve_adjoint(g: np.ndarray, C: int, N: int) -> np.ndarray:
    g = np.asarray(g, dtype=np.float64)
    gz = np.empty_like(g)
    col = 0
    for wk, M in psi_phi_blocks(C, N):
        n = len(wk)
        rhs = g[..., col:col + n].reshape(-1, n).T
        sol = solve_triangular(M, rhs, lower=True, trans="T")
        gz[..., col:col + n] = sol.T.reshape(g.shape[:-1] + (n,))
        col += n
    return psi_adjoint(gz, C, N)


def phi_expand_flat(alpha: np.ndarray, C: int, N: int) -> np.ndarray:
    """sum_l alpha_l phi(l) as a flat truncated tensor (the left side of eq-linearsystem)."""
    alpha = np.asarray(alpha, dtype=np.float64)
    S = sum(C ** k for k in range(1, N + 1))
    out = np.zeros(alpha.shape[:-1] + (S,))
    for j, w in enumerate(lyndon_words(C, N)):
        for u, c in phi(w).items():
            out[..., _flat_index(u, C)] += c * alpha[..., j]
    return out
