"""bench.py's multi-process plumbing on CPU: `--gpus N` launches N ranks itself (torchrun on
127.0.0.1), the ranks rendezvous, time, reduce max-over-ranks and rank 0 prints one JSON line with
n_gpus = N; a --gpus that disagrees with WORLD_SIZE is refused.  --dry-run replaces the kernels with
a CPU stub (no oracle either) so this runs without a GPU."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None, timeout=300):
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                          env=e, timeout=timeout, cwd=ROOT)


def _json_lines(out):
    return [json.loads(l) for l in out.splitlines() if l.startswith("{")]


@pytest.mark.parametrize("scaling", ["weak", "strong"])
def test_bench_self_launches_world2_gloo(scaling):
    r = _run(["--gpus", "2", "--backend", "gloo", "--dry-run", "--steps", "4", "--warmup", "3", "--scaling", scaling])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1, r.stdout  # rank 0 only
    assert lines[0]["n_gpus"] == 2 and lines[0]["backend"] == "gloo" and lines[0]["scaling"] == scaling


def test_bench_refuses_mismatched_world():
    r = _run(["--gpus", "4", "--dry-run", "--steps", "3"], env={"WORLD_SIZE": "2", "RANK": "0"})
    assert r.returncode != 0
    assert "WORLD_SIZE" in (r.stderr + r.stdout)


@pytest.mark.gpu
@pytest.mark.parametrize("config,scaling", [("c2", "strong"), ("c5", "weak")])
def test_bench_world2_real_kernels_one_gpu(config, scaling):
    """The N-rank path of bench.py with the real kernels: two ranks share cuda:0 over gloo
    (SIGB200_BENCH_SHARE_GPU=1; the multi-GPU NCCL box is not available to this build).  Checks
    that the arm runs end to end (batch shards, or c5's time chunks with the all-gather and ordered
    fold) and rank 0 prints one line with n_gpus = 2 -- not a measurement of two GPUs."""
    r = _run(["--gpus", "2", "--backend", "gloo", "--config", config, "--scaling", scaling, "--steps", "3",
              "--warmup", "3", "--no-configs", "--no-cpu-baseline"], env={"SIGB200_BENCH_SHARE_GPU": "1"}, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1, r.stdout
    ln = lines[0]
    assert ln["n_gpus"] == 2 and ln["value"] > 0 and ln["gpu_launches"] > 0
    assert ln["scaling"] == ("strong" if config == "c5" else scaling)
