"""Error metrics for GPU-vs-oracle parity (reading R9 / SURVEY Z9).

Forward: norm-wise relative error per (path, level): ||gpu_k - ref_k||_inf / ||ref_k||_inf,
maximised over paths and levels (a level whose reference is exactly zero is compared in
absolute terms against 1e-6).  Backward: per path and output tensor, ||gpu - ref||_inf / ||ref||_inf.
Bars (BASELINE.json north_star): 1e-4 forward, 5e-4 backward.
"""
import numpy as np

FWD_TOL = 1e-4
BWD_TOL = 5e-4


def level_rel_err(gpu, ref, C, N):
    gpu = np.asarray(gpu, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    worst = 0.0
    off = 0
    for k in range(1, N + 1):
        n = C ** k
        g = gpu[..., off:off + n].reshape(-1, n)
        r = ref[..., off:off + n].reshape(-1, n)
        num = np.max(np.abs(g - r), axis=1)
        den = np.max(np.abs(r), axis=1)
        e = np.where(den > 0, num / np.where(den > 0, den, 1), num / 1e-6)
        worst = max(worst, float(np.max(e)) if e.size else 0.0)
        off += n
    return worst


def block_rel_err(gpu, ref, blocks):
    """blocks: list of (start, stop) column ranges (e.g. Lyndon degree blocks)."""
    gpu = np.asarray(gpu, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    worst = 0.0
    for a, b in blocks:
        g = gpu[..., a:b].reshape(-1, b - a)
        r = ref[..., a:b].reshape(-1, b - a)
        num = np.max(np.abs(g - r), axis=1)
        den = np.max(np.abs(r), axis=1)
        e = np.where(den > 0, num / np.where(den > 0, den, 1), num / 1e-6)
        worst = max(worst, float(np.max(e)) if e.size else 0.0)
    return worst


def path_rel_err(gpu, ref):
    """per leading index (path): ||gpu - ref||_inf / ||ref||_inf, maximised."""
    gpu = np.asarray(gpu, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    g = gpu.reshape(gpu.shape[0], -1)
    r = ref.reshape(ref.shape[0], -1)
    num = np.max(np.abs(g - r), axis=1)
    den = np.max(np.abs(r), axis=1)
    e = np.where(den > 0, num / np.where(den > 0, den, 1), num / 1e-6)
    return float(np.max(e))
