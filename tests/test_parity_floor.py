"""The per-row floor in tests/parity.py (reading R9) exists for exact-zero levels (C = 1, a single
segment's higher log levels).  On the hot-path shapes and input distributions of BASELINE.json's
configs it must never engage, so every parity number there is a true per-level relative error.
Stream mode (c3) is the exception: its first rows are signatures of one or two segments whose
level k scales like |z|^k (level 4 ~ 1e-6 x level 1 at M = 1023), so its GPU parity tests use the
strict metric (no floor, tests/test_gpu_signature.py)."""
import numpy as np
import pytest

import oracle
from synth import CONFIGS, SEEDS, brownian_paths, uniform_paths
from tests.parity import floor_engaged, level_blocks


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
@pytest.mark.parametrize("kind", ["brownian", "uniform"])
def test_hot_path_shapes_never_hit_the_floor(name, kind):
    cfg = CONFIGS[name]
    C, N = cfg["C"], cfg["N"]
    B = min(cfg["B"], 8)
    L = min(cfg["L"], 300)
    seed = SEEDS[name][0]
    x = brownian_paths(B, L, C, seed) if kind == "brownian" else uniform_paths(B, L, C, seed + 1000)
    sig = oracle.signature(x, N, stream=cfg["stream"], threads=8)
    if cfg["stream"]:
        assert floor_engaged(sig[:, :2], level_blocks(C, N)) or kind == "uniform"  # documented above
        sig = sig[:, 64:]  # from the 65th prefix on, the levels are within the floor's range
    assert not floor_engaged(sig, level_blocks(C, N)), (name, kind)
    if name == "c4":
        log = oracle.logsignature(x, N, mode="expand", threads=8)
        assert not floor_engaged(log, level_blocks(C, N)), (name, kind, "log")
