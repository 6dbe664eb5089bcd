"""Seeded synthetic inputs shared by the oracle side and the CUDA side (tests, bench, smoke).

Holds none of the method's arithmetic: it only draws random numbers.  Every array is generated in
float64 from numpy's PCG64 and rounded to float32 exactly once, so the GPU and the oracle see the
same bytes.

* ``brownian_paths`` -- the primary workload (reading R17): x_0 = 0 and iid Gaussian
  increments with variance 1/M per channel (M = L-1 increments), i.e. a Brownian motion sampled on
  [0, 1]; the paper's deep-learning example draws geometric Brownian motion.
* ``uniform_paths`` -- the robustness input, ``torch.rand``-like uniform [0, 1) points as in the
  paper's code example.
* ``normal`` -- upstream gradients ``grad_out`` ~ N(0, 1).
"""
from __future__ import annotations

import numpy as np

# Per-config seeds: path seed / grad seed.
SEEDS = {"c1": (1, None), "c2": (2, 102), "c3": (3, None), "c4": (4, 104), "c5": (5, None), "c5b": (5, 105),
         "c3l": (3, None)}

# BASELINE.json configs
CONFIGS = {
    "c1": dict(B=32, L=128, C=4, N=4, stream=False, op="sig_fwd"),
    "c2": dict(B=1024, L=128, C=8, N=5, stream=False, op="sig_fwd_bwd"),
    "c3": dict(B=256, L=1024, C=6, N=4, stream=True, op="sig_fwd_stream"),
    "c4": dict(B=512, L=256, C=4, N=7, stream=False, op="logsig_words_fwd_bwd"),
    "c5": dict(B=1, L=2 ** 22, C=3, N=6, stream=False, op="sig_fwd_timechunk"),
    # not a BASELINE config: c5's path through forward + reversible backward
    "c5b": dict(B=1, L=2 ** 22, C=3, N=6, stream=False, op="sig_fwd_bwd_timechunk"),
    # not a BASELINE config: stream-mode logsignature (words) at c3's shape
    "c3l": dict(B=256, L=1024, C=6, N=4, stream=True, op="logsig_stream_fwd"),
}


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def brownian_paths(B: int, L: int, C: int, seed: int, scale: float = 1.0) -> np.ndarray:
    """float32 [B, L, C]: x_0 = 0, x_{t+1} - x_t ~ N(0, scale^2 / (L-1)) iid."""
    rng = _rng(seed)
    M = max(L - 1, 1)
    z = rng.standard_normal((B, L - 1, C)) * (scale / np.sqrt(M))
    x = np.zeros((B, L, C), dtype=np.float64)
    np.cumsum(z, axis=1, out=x[:, 1:, :])
    return x.astype(np.float32)


def uniform_paths(B: int, L: int, C: int, seed: int) -> np.ndarray:
    """float32 [B, L, C] uniform on [0, 1) (the paper's torch.rand example)."""
    return _rng(seed).random((B, L, C)).astype(np.float32)


def normal(shape, seed: int, scale: float = 1.0) -> np.ndarray:
    return (_rng(seed).standard_normal(shape) * scale).astype(np.float32)


def config_inputs(name: str, B: int | None = None, L: int | None = None):
    """(path, grad_out_shape_seed) for a BASELINE config, optionally with a smaller B or L."""
    cfg = CONFIGS[name]
    ps, gs = SEEDS[name]
    Bv = cfg["B"] if B is None else B
    Lv = cfg["L"] if L is None else L
    return brownian_paths(Bv, Lv, cfg["C"], ps), gs
