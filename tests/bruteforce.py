"""Independent brute-force references used only to PIN the oracle (not the oracle itself).

* ``iterated_integrals``: the signature definition (eq-signaturedef) evaluated exactly for
  the piecewise-affine interpolant (dfn-stream-sig).  Assign each of the k ordered times
  t_1 < ... < t_k to the segment it falls in: the segment indices s_1 <= ... <= s_k are
  non-decreasing, each segment contributes its (constant) derivative z_s, and r times falling in
  the same segment contribute the volume 1/r! of the ordered r-simplex.  So
      S_k[w] = sum_{s_1<=...<=s_k} prod_m z_{s_m}[w_m] / prod_runs r!.
  This never uses Chen's identity or the exp-then-[x] recursion the oracle uses.
* ``levy_area``: the textbook shoelace formula for the area of a piecewise-linear path.
* ``finite_difference``: central differences.
"""
from __future__ import annotations

import itertools
import math
from functools import reduce

import numpy as np


def iterated_integrals(path: np.ndarray, N: int) -> np.ndarray:
    x = np.asarray(path, dtype=np.float64)
    z = np.diff(x, axis=0)  # [M, C]
    M, C = z.shape
    out = []
    for k in range(1, N + 1):
        acc = np.zeros((C,) * k)
        for s in itertools.combinations_with_replacement(range(M), k):
            runs = [len(list(g)) for _, g in itertools.groupby(s)]
            weight = 1.0 / math.prod(math.factorial(r) for r in runs)
            acc += weight * reduce(np.multiply.outer, [z[i] for i in s])
        out.append(acc.reshape(-1))
    return np.concatenate(out)


def levy_area(path: np.ndarray) -> np.ndarray:
    """A[i,j] = 1/2 sum_{s<t} (z_s[i] z_t[j] - z_t[i] z_s[j])."""
    z = np.diff(np.asarray(path, dtype=np.float64), axis=0)
    M, C = z.shape
    A = np.zeros((C, C))
    for s in range(M):
        for t in range(s + 1, M):
            A += 0.5 * (np.outer(z[s], z[t]) - np.outer(z[t], z[s]))
    return A


def finite_difference(f, x: np.ndarray, h: float = 1e-6) -> np.ndarray:
    """Central differences of a scalar function f at x (float64)."""
    x = np.array(x, dtype=np.float64)
    g = np.zeros_like(x)
    it = np.nditer(x, flags=["multi_index"])
    for _ in it:
        i = it.multi_index
        xp = x.copy()
        xm = x.copy()
        xp[i] += h
        xm[i] -= h
        g[i] = (f(xp) - f(xm)) / (2 * h)
    return g


def rel_err(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = max(np.max(np.abs(b)), 1e-300)
    return float(np.max(np.abs(a - b)) / den)
