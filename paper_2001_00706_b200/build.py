"""Build libsig.so (the C-ABI library of include/sig.h) in-tree for sm_100a.

    python -m paper_2001_00706_b200.build [-j N] [--force]

Compiles every translation unit under csrc/ with
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC
in parallel, then links paper_2001_00706_b200/libsig.so with the CUDA runtime linked statically
(the library has no torch dependency; the Python binding only passes pointers and streams).
"""
from __future__ import annotations

import argparse
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
# SIGB200_BUILD_TAG builds a variant (extra -D flags from SIGB200_EXTRA_FLAGS) into libsig_<tag>.so
_TAG = os.environ.get("SIGB200_BUILD_TAG", "")
OBJ = os.path.join(HERE, "build_obj" + (f"_{_TAG}" if _TAG else ""))
LIB = os.path.join(HERE, f"libsig_{_TAG}.so" if _TAG else "libsig.so")
_EXTRA = os.environ.get("SIGB200_EXTRA_FLAGS", "").split()
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "--extended-lambda", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
         "-Xptxas", "-warn-spills"]


def _sources():
    srcs = [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC)) if f.endswith(".cu") or f.endswith(".cpp")]
    return srcs


def _headers_mtime():
    ts = [os.path.getmtime(os.path.join(CSRC, f)) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h", ".py"))]
    ts.append(os.path.getmtime(os.path.join(HERE, "..", "include", "sig.h")))
    return max(ts)


def _compile(src: str, force: bool, hdr_t: float) -> tuple[str, str]:
    obj = os.path.join(OBJ, os.path.basename(src) + ".o")
    if not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), hdr_t):
        return obj, ""
    cmd = [NVCC, *ARCH, *FLAGS, *_EXTRA, "-c", src, "-o", obj]
    if src.endswith(".cpp"):
        cmd = [NVCC, "-x", "c++", *FLAGS[:4], "-Xcompiler", "-fPIC", "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr


def build(force: bool = False, jobs: int | None = None, verbose: bool = False) -> str:
    sys.path.insert(0, CSRC)
    import gen_instances  # noqa: E402

    gen_instances.main()
    sys.path.pop(0)
    os.makedirs(OBJ, exist_ok=True)
    hdr_t = _headers_mtime()
    srcs = _sources()
    jobs = jobs or max(1, min(len(srcs), os.cpu_count() or 4))
    with ThreadPoolExecutor(max_workers=jobs) as ex:
        results = list(ex.map(lambda s: _compile(s, force, hdr_t), srcs))
    objs = [o for o, _ in results]
    if verbose:
        for o, log in results:
            if log.strip():
                print(os.path.basename(o), log, file=sys.stderr)
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-j", type=int, default=None)
    ap.add_argument("-v", action="store_true")
    a = ap.parse_args()
    print(build(force=a.force, jobs=a.j, verbose=a.v))
