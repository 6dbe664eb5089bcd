"""Error metrics for GPU-vs-oracle parity (reading R9 / SURVEY Z9).

Forward: norm-wise relative error per (path, level): ||gpu_k - ref_k||_inf / ||ref_k||_inf,
maximised over paths and levels.  A level whose reference norm is below 1e-4 x the largest level
norm of the same row (exact zeros such as the higher log levels of a single segment, or levels
wiped out by cancellation) is judged against that floor instead (reading R9).  Backward: per path and output tensor, ||gpu - ref||_inf / ||ref||_inf.
Bars (BASELINE.json north_star): 1e-4 forward, 5e-4 backward.
"""
import numpy as np

FWD_TOL = 1e-4
BWD_TOL = 5e-4


FLOOR_REL = 1e-4


def floor_engaged(ref, blocks) -> bool:
    """True when some (row, block) reference norm is below FLOOR_REL x its row's largest block norm,
    i.e. when _blocks_err would judge that block against the floor instead of its own norm."""
    r = np.asarray(ref, dtype=np.float64)
    r = r.reshape(-1, r.shape[-1])
    norms = np.stack([np.max(np.abs(r[:, a:b]), axis=1) for a, b in blocks], axis=1)
    return bool(np.any(norms < FLOOR_REL * np.max(norms, axis=1, keepdims=True)))


def level_blocks(C, N):
    blocks, off = [], 0
    for k in range(1, N + 1):
        blocks.append((off, off + C ** k))
        off += C ** k
    return blocks


def _blocks_err(gpu, ref, blocks, strict=False):
    gpu = np.asarray(gpu, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    W = gpu.shape[-1]
    g = gpu.reshape(-1, W)
    r = ref.reshape(-1, W)
    norms = np.stack([np.max(np.abs(r[:, a:b]), axis=1) for a, b in blocks], axis=1)  # [rows, nblocks]
    floor = (0.0 if strict else FLOOR_REL) * np.max(norms, axis=1)
    worst = 0.0
    for j, (a, b) in enumerate(blocks):
        num = np.max(np.abs(g[:, a:b] - r[:, a:b]), axis=1)
        den = np.maximum(norms[:, j], floor)
        den = np.where(den > 0, den, 1e-30)
        worst = max(worst, float(np.max(num / den)) if num.size else 0.0)
    return worst


def level_rel_err(gpu, ref, C, N, strict=False):
    """strict: every (row, level) against its own norm (no floor) -- used where levels of one row span
    many orders of magnitude legitimately (the first rows of stream mode)."""
    return _blocks_err(gpu, ref, level_blocks(C, N), strict)


def block_rel_err(gpu, ref, blocks):
    """blocks: list of (start, stop) column ranges (e.g. Lyndon degree blocks)."""
    return _blocks_err(gpu, ref, blocks)


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
