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
