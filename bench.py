"""Benchmark of the Signatory hot path on B200 (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2]

Default workload = BASELINE.json's metric configuration c2: signature forward + reversible backward,
B = 1024 paths/GPU, L = 128, C = 8, depth N = 5, seeded Brownian paths (synth/), float32.  A
"step" is one pass of the whole hot path over one batch: sig_signature then sig_signature_backward
with an upstream gradient grad_out ~ N(0,1).  With --gpus N > 1 (torchrun, one process per GPU,
NCCL) every rank processes its own batch of B paths (batch sharding: the paths are independent,
no data-path collective, "weak" scaling); timing is CUDA events on the launching stream,
barrier + synchronize around the timed region, max over ranks.

Other keys: roofline (dominant kernel = the reversible backward, FP32 FMA "alu"-bound, see
DESIGN.md "Roofline"), cpu_baseline (the float64 oracle on the host cores, bounded sample), e2e
(the same step through the C ABI from pinned host buffers: H2D of path + grad_out, D2H of
grad_path inside the timed region), clocks (NVML samples during the timed region), gpu_launches
(library launch counter).  --impl reference times the oracle itself (the reference arm).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth import CONFIGS, SEEDS, brownian_paths, normal  # noqa: E402

METRIC = "signature fwd+bwd paths/sec (B=1024,L=128,C=8,N=5) at 1/2/4/8 B200; % FP32 peak"
UNIT = "paths/s"


def fused_cost(d: int, N: int) -> int:
    """F(d, N) = d(N-1) + sum_{k=1}^N sum_{i=2}^k d^i  (eq-fusedresult)."""
    return d * (N - 1) + sum(d ** i for k in range(1, N + 1) for i in range(2, k + 1))


def alg_flops(op: str, B: int, M: int, C: int, N: int) -> float:
    """Algorithmic FLOPs: 2F per increment forward,
    4F(C,N) + 2F(C,N-1) per increment backward."""
    if op == "fwd":
        return 2.0 * fused_cost(C, N) * M * B
    return (4.0 * fused_cost(C, N) + 2.0 * fused_cost(C, N - 1)) * M * B


def fp32_peak_tflops() -> tuple[float, str, float | None]:
    """FP32 FMA peak: 148 SMs x 128 FP32 lanes x 2 FLOP x 1.965 GHz (max SM clock in
    MEASURED_PEAKS.json) = 74.45 TFLOP/s.  MEASURED_PEAKS.json carries no FP32 figure; DESIGN.md
    derives this denominator from the guide's unit counts and clocks.  The third value is the
    FFMA microbenchmark's measured peak on this pool (profiles/fp32_peak.json), reported beside it."""
    mhz = 1965.0
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        mhz = float(mp.get("sm_max_mhz", mhz))
    except Exception:
        pass
    meas = None
    try:
        meas = float(json.load(open(os.path.join(ROOT, "profiles", "fp32_peak.json")))["tflops"])
    except Exception:
        pass
    return (148 * 128 * 2 * mhz * 1e6 / 1e12, f"148 SM x 128 lanes x 2 x {mhz:.0f} MHz (derived, DESIGN.md)", meas)


class ClockSampler:
    """NVML samples of the SM clock and the active clock-event reasons during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------------------------------------
def cpu_baseline(cfg_name: str, seconds: float = 15.0) -> dict:
    """The float64 oracle (test infrastructure, as it stands) on the host cores: a bounded sample
    of the same workload (the first paths of the same seeded batch; for the single long path of c5
    a prefix of it, scaled to whole paths), threads = all cores."""
    import oracle

    cfg = CONFIGS[cfg_name]
    C, N, L = cfg["C"], cfg["N"], cfg["L"]
    cores = len(os.sched_getaffinity(0)) or 1
    ps, gs = SEEDS[cfg_name]
    if cfg_name in ("c5", "c5b"):
        Ls = 2 ** 17 + 1
        x = brownian_paths(1, L, C, ps)[:, :Ls]
        t0 = time.perf_counter()
        _oracle_step(oracle, cfg_name, x, gs, 1)
        dt = time.perf_counter() - t0
        frac = (Ls - 1) / (L - 1)
        return {"value": frac / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
                "sample": f"first {Ls} of {L} points of the c5 path (float64 C oracle, 1 thread: the scan is "
                          f"sequential), {dt:.1f} s, scaled by {frac:.4f}"}
    # size the sample from a 1-path probe so the run stays within ~`seconds`
    x1 = brownian_paths(1, L, C, ps)
    t0 = time.perf_counter()
    _oracle_step(oracle, cfg_name, x1, gs, 1)
    per_path = max(time.perf_counter() - t0, 1e-6)
    n = int(max(1, min(cfg["B"], seconds * cores / per_path)))
    n = max(cores, (n // cores) * cores) if n >= cores else n
    x = brownian_paths(cfg["B"], L, C, ps)[:n]
    t0 = time.perf_counter()
    _oracle_step(oracle, cfg_name, x, gs, cores)
    dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": UNIT, "cores": min(cores, n), "kind": "oracle",
            "sample": f"{n} of {cfg['B']} paths of {cfg_name} ({cfg['op']}, float64 C oracle, {min(cores, n)} threads), "
                      f"{dt:.1f} s"}


def _oracle_step(oracle, cfg_name, x, gs, threads):
    cfg = CONFIGS[cfg_name]
    C, N = cfg["C"], cfg["N"]
    S = sum(C ** k for k in range(1, N + 1))
    if cfg["op"] in ("sig_fwd_bwd", "sig_fwd_bwd_timechunk"):
        g = normal((x.shape[0], S), gs)
        oracle.signature_vjp(g, x, N, threads=threads)  # includes the forward it needs
    elif cfg["op"] == "logsig_words_fwd_bwd":
        from oracle import lyndon
        g = normal((x.shape[0], lyndon.witt(C, N)), gs)
        oracle.logsignature_vjp(g, x, N, mode="words", threads=threads)
    elif cfg["op"] == "logsig_stream_fwd":
        oracle.logsignature(x, N, mode="words", stream=True, threads=threads)
    else:
        oracle.signature(x, N, stream=cfg["stream"], threads=threads)


# ------------------------------------------------------------------------------------------------
def run_reference(args, rank: int, world: int):
    """Reference arm: the float64 oracle, as it stands, on the host cores."""
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    import oracle

    cores = len(os.sched_getaffinity(0)) or 1
    if args.config in ("c5", "c5b"):  # one long path: each step is a bounded prefix, scaled to whole paths
        Ls = 2 ** 16 + 1
        x = brownian_paths(1, cfg["L"], cfg["C"], SEEDS["c5"][0])[:, :Ls]
        n = (Ls - 1) / (cfg["L"] - 1)
        sample = f"first {Ls} points of the c5 path per step (scaled), float64 C oracle, 1 thread"
        used = 1
    else:
        n = min(cfg["B"], max(cores, 16))
        x = brownian_paths(cfg["B"], cfg["L"], cfg["C"], SEEDS[args.config][0])[:n]
        sample = f"{n} of {cfg['B']} paths per step, float64 C oracle, {min(cores, n)} threads"
        used = min(cores, n)
    for _ in range(args.warmup):
        _oracle_step(oracle, args.config, x[: max(1, min(cores, x.shape[0]))], SEEDS[args.config][1], cores)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        _oracle_step(oracle, args.config, x, SEEDS[args.config][1], cores)
        ts.append(time.perf_counter() - t0)
    ms = 1000 * float(np.mean(ts))
    val = n / (ms / 1000)
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": _config_dict(args.config, world),
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": used, "kind": "oracle", "sample": sample},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _config_dict(name, world, scaling="weak", B=None, l2=None):
    cfg = CONFIGS[name]
    B = B or cfg["B"]
    if name in ("c5", "c5b"):
        par = f"time-chunk x{world} (NCCL all-gather + ordered fold)" if world > 1 else "single GPU"
        bdesc = "B=1"
    elif scaling == "strong":
        par = f"batch-shard x{world}, global batch {B} (rank r: dist.batch_bounds)" if world > 1 else "single GPU"
        bdesc = f"B={B} global"
    else:
        par = f"batch-shard x{world}, {B} paths per GPU" if world > 1 else "single GPU"
        bdesc = f"B={B}/GPU"
    return {"workload": f"{name}: {cfg['op']} {bdesc} L={cfg['L']} C={cfg['C']} N={cfg['N']}"
                        f"{' stream' if cfg['stream'] else ''}, Brownian",
            "B_per_gpu" if scaling != "strong" else "B_global": B, "L": cfg["L"], "C": cfg["C"],
            "depth": cfg["N"], "stream": cfg["stream"], "parallelism": par, "scaling": scaling,
            "l2": l2 or ("per-step working set > 126 MB L2 (grad_out + signature 307 MB); no flush needed"
                         if name == "c2" else "see DESIGN.md")}


# ------------------------------------------------------------------------------------------------
L2_BYTES = 126 * 2 ** 20


class Workload:
    """One BASELINE config as a benchmark step.  step(ev) runs one step on the device (ev: list of
    (label, event) marks for the live per-segment split, or None); e2e_step() runs it from pinned
    host buffers; units = paths this rank processes per step.

    scaling: "weak" -- every rank its own batch of B paths (B = the config's, or --batch);
             "strong" -- one global batch of B paths, rank r takes [rB/G, (r+1)B/G) (dist.batch_bounds);
    c5 is always time-chunked over the ranks (one path per step for the whole job)."""

    def __init__(self, name, rank, world, dev, scaling="weak", batch=None):
        import torch

        import paper_2001_00706_b200 as sb
        from paper_2001_00706_b200 import dist as sdist

        self.sb, self.torch, self.dev, self.name = sb, torch, dev, name
        cfg = CONFIGS[name]
        self.cfg = cfg
        self.L, self.C, self.N = cfg["L"], cfg["C"], cfg["N"]
        self.S = sb.sig_signature_channels(self.C, self.N)
        ps, gs = SEEDS[name]
        self.world, self.rank = world, rank
        self.scaling = "strong" if name in ("c5", "c5b") else scaling
        B0 = int(batch) if batch else cfg["B"]
        if name in ("c5", "c5b"):
            full = brownian_paths(1, self.L, self.C, ps)  # the one long path, time-chunked over ranks
            a, b = sdist.time_chunk_bounds(self.L, world, rank)
            self.x_np = np.ascontiguousarray(full[:, a:b])
            self.M = b - a - 1
            self.B = 1
            self.B_global = 1
            self.units = 1.0 / world  # one path per step for the whole job
            self.gsl = slice(0, 1)
        elif self.scaling == "strong":
            lo, hi = sdist.batch_bounds(B0, world, rank)
            self.x_np = np.ascontiguousarray(brownian_paths(B0, self.L, self.C, ps)[lo:hi])
            self.B, self.B_global, self.M = hi - lo, B0, self.L - 1
            self.units = float(self.B)
            self.gsl = slice(lo, hi)
        else:
            self.x_np = brownian_paths(B0, self.L, self.C, ps + 7919 * rank)
            self.B, self.B_global, self.M = B0, B0 * world, self.L - 1
            self.units = float(B0)
            self.gsl = slice(0, B0)
        self.x = torch.from_numpy(self.x_np).to(dev)
        self.g = None
        gseed = (gs or 0) + (7919 * rank if self.scaling == "weak" else 0)
        if cfg["op"] in ("sig_fwd_bwd", "sig_fwd_bwd_timechunk"):
            self.g_np = normal((B0, self.S), gseed)[self.gsl]
        elif cfg["op"] == "logsig_words_fwd_bwd":
            self.g_np = normal((B0, sb.sig_logsignature_channels(self.C, self.N, "words")), gseed)[self.gsl]
        else:
            self.g_np = None
        if self.g_np is not None:
            self.g_np = np.ascontiguousarray(self.g_np)
            self.g = torch.from_numpy(self.g_np).to(dev)
        self.stream = torch.cuda.current_stream(dev)
        # per-step working set: inputs larger than L2 need no flush between timed steps
        ws = self.x.numel() * 4 + (self.g.numel() * 4 if self.g is not None else 0)
        if cfg["op"] == "sig_fwd_bwd":
            ws += self.B * self.S * 4 * 2
        elif cfg["op"] == "sig_fwd_stream":
            ws += self.B * self.M * self.S * 4
        elif cfg["op"] == "logsig_words_fwd_bwd":
            ws += self.B * self.S * 4 * 4
        elif cfg["op"] == "logsig_stream_fwd":
            self.W = sb.sig_logsignature_channels(self.C, self.N, "words")
            ws += self.B * self.M * (self.S + self.W) * 4
        self.working_set = ws
        self.flush = ws <= L2_BYTES
        self.graph = name == "c1"  # latency-bound: replay the step from a CUDA graph (time_workload)
        self.l2 = (f"per-step working set {ws / 1e6:.0f} MB > 126 MB L2; no flush needed" if not self.flush else
                   f"per-step working set {ws / 1e6:.1f} MB < L2: L2 flushed (256 MB write) before every timed step, "
                   f"outside the per-step events")

    def _run(self, x, g, ev):
        sb, N, torch = self.sb, self.N, self.torch

        def mark(lab):
            if ev is not None:
                e = torch.cuda.Event(enable_timing=True)
                e.record(self.stream)
                ev.append((lab, e))

        op = self.cfg["op"]
        mark("start")
        if op == "sig_fwd_bwd":
            out = sb.sig_signature(x, N)
            mark("fwd")
            res, _ = sb.sig_signature_backward(g, x, out, N)
            mark("bwd")
        elif op == "logsig_words_fwd_bwd":
            out, sig = sb.sig_logsignature(x, N, "words", return_signature=True)
            mark("fwd")
            res, _ = sb.sig_logsignature_backward(g, x, sig, N, "words")
            mark("bwd")
        elif op == "logsig_stream_fwd":
            res = sb.sig_logsignature(x, N, "words", stream=True)
            mark("fwd")
        elif op == "sig_fwd_timechunk":
            from paper_2001_00706_b200 import dist as sdist

            res = sdist.dist_signature_timechunk(x, N) if self.world > 1 else sb.sig_signature(x, N)
            mark("fwd")
        elif op == "sig_fwd_bwd_timechunk":
            from paper_2001_00706_b200 import dist as sdist

            if self.world > 1:
                sig, parts = sdist.dist_signature_timechunk(x, N, return_parts=True)
                mark("fwd")
                res = sdist.dist_signature_timechunk_backward(g, x, parts, N)
            else:
                # the forward keeps the chunk states the time-parallel backward starts from
                # (sig_signature_save), so the backward does not recompute the chunk signatures
                out, saved = sb.sig_signature_save(x, N)
                mark("fwd")
                res, _ = sb.sig_signature_backward_saved(g, x, out, saved, N)
            mark("bwd")
        else:
            res = sb.sig_signature(x, N, stream=self.cfg["stream"])
            mark("fwd")
        return res

    def step(self, ev=None):
        return self._run(self.x, self.g, ev)

    def prepare_e2e(self):
        torch = self.torch
        self.xh = torch.from_numpy(self.x_np).pin_memory()
        self.gh = torch.from_numpy(self.g_np).pin_memory() if self.g_np is not None else None
        self.xd = torch.empty_like(self.x)
        self.gd = torch.empty_like(self.g) if self.g is not None else None
        res = self.step()
        self.resh = torch.empty(res.shape, dtype=res.dtype).pin_memory()
        self.h2d = self.xh.numel() * 4 + (self.gh.numel() * 4 if self.gh is not None else 0)
        self.d2h = self.resh.numel() * 4
        # c2 is transfer-bound (153 MB of grad_out per step): the native host-buffer entry point
        # sig_signature_fwd_bwd_host overlaps the copies of one batch slice with the kernels of
        # another.  c4 moves 9 MB and is kernel-bound; slicing its batch only costs kernel efficiency.
        self.pipe = "native" if self.cfg["op"] == "sig_fwd_bwd" else None

    def e2e_step(self):
        if self.pipe is not None:
            # one C-ABI call with host buffers: H2D of slice k+1 and D2H of slice k-1 overlap the
            # kernels of slice k
            self.sb.sig_signature_fwd_bwd_host(self.xh, self.gh, self.N, chunks=4, grad_path_h=self.resh,
                                               device=self.x.device)
            return
        self.xd.copy_(self.xh, non_blocking=True)
        if self.gh is not None:
            self.gd.copy_(self.gh, non_blocking=True)
        res = self._run(self.xd, self.gd, None)
        self.resh.copy_(res, non_blocking=True)

    def roofline(self, seg_ms, ms_step):
        """Dominant kernel's roofline from the live per-segment CUDA-event times."""
        C, N, M, B = self.C, self.N, self.M, self.B
        peak, peak_src, peak_meas = fp32_peak_tflops()
        op = self.cfg["op"]
        try:
            traffic = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json"))).get(self.name, {})
        except Exception:
            traffic = {}
        meas = (lambda a: {"peak_measured": peak_meas, "frac_of_measured": a / peak_meas} if peak_meas else {})
        if op in ("sig_fwd_bwd", "logsig_words_fwd_bwd", "sig_fwd_bwd_timechunk"):
            f_fwd = alg_flops("fwd", B, M, C, N)
            f_bwd = alg_flops("bwd", B, M, C, N)
            ach = f_bwd / (seg_ms["bwd"] / 1000) / 1e12
            kern = {"sig_fwd_bwd": "sig_bwd2p_kernel (reversible backward, sibling prefixes packed per FFMA2)",
                    "logsig_words_fwd_bwd": "sig_logsignature_backward call = logsig_bwd_kernel + sig_bwd_kernel "
                                            "(sig-bwd FLOPs only)",
                    "sig_fwd_bwd_timechunk": "time-parallel reversible backward (chunk signatures, ordered scans, "
                                             "chunk-end VJPs, sig_bwd_kernel over all chunks)"}[op]
            r = {"bound": "alu", "kernel": kern, "achieved": ach, "peak": peak, "unit": "TFLOP/s",
                 "frac": ach / peak, "traffic": traffic.get("dominant_kernel"), "peak_source": peak_src,
                 "kernel_ms": seg_ms["bwd"], "step_share": seg_ms["bwd"] / (seg_ms["fwd"] + seg_ms["bwd"]),
                 "fwd": {"kernel_ms": seg_ms["fwd"], "achieved": f_fwd / (seg_ms["fwd"] / 1000) / 1e12,
                         "frac": f_fwd / (seg_ms["fwd"] / 1000) / 1e12 / peak},
                 "step_frac": (f_fwd + f_bwd) / (ms_step / 1000) / 1e12 / peak}
            r.update(meas(ach))
            return r
        if op == "logsig_stream_fwd":
            hbm = 6543.7
            try:
                hbm = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
            except Exception:
                pass
            # algorithmic bytes: the path read, every prefix signature written once (the state the
            # C ABI keeps for the backward, B M S floats) and the words written (B M w floats).  As
            # built the two kernels also read the signatures back (K1 stream writes them, K4 reads
            # them): reported as bytes_as_built beside it.
            rows = B * M
            nbytes = (rows * self.S + rows * self.W) * 4 + B * self.L * C * 4
            built = nbytes + rows * self.S * 4
            ach = nbytes / (seg_ms["fwd"] / 1000) / 1e9
            return {"bound": "hbm", "kernel": "sig_fwd_stream_kernel + logsig_rows_t_kernel (stream logsignature; "
                    "algorithmic bytes = path + signature rows + words)", "achieved": ach, "peak": hbm,
                    "unit": "GB/s", "frac": ach / hbm, "traffic": traffic.get("dominant_kernel"),
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs", "kernel_ms": seg_ms["fwd"],
                    "bytes_as_built": built, "as_built_gbs": built / (seg_ms["fwd"] / 1000) / 1e9,
                    "output_gbs": rows * self.W * 4 / (seg_ms["fwd"] / 1000) / 1e9}
        if op == "sig_fwd_stream":
            hbm = 6543.7
            try:
                hbm = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
            except Exception:
                pass
            nbytes = B * M * self.S * 4 + B * self.L * C * 4  # written prefixes + read path
            ach = nbytes / (seg_ms["fwd"] / 1000) / 1e9
            return {"bound": "hbm", "kernel": "sig_fwd_stream_kernel (stream=True, staged rows + TMA bulk stores)",
                    "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                    "traffic": traffic.get("dominant_kernel"), "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                    "kernel_ms": seg_ms["fwd"]}
        f = alg_flops("fwd", B, M, C, N)
        ach = f / (seg_ms["fwd"] / 1000) / 1e12
        r = {"bound": "alu",
             "kernel": "sig_fwd_kernel (+ ordered chunk fold" + (", NCCL all-gather)" if self.world > 1 else ")"),
             "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
             "traffic": traffic.get("dominant_kernel"), "peak_source": peak_src, "kernel_ms": seg_ms["fwd"]}
        r.update(meas(ach))
        return r


def bind_gpu_local_cpus(index: int):
    """Pin this process to the CPUs NVML reports as local to GPU `index` before any pinned host
    buffer is allocated (first touch then places the pages on the GPU's NUMA node; on a remote node
    the host<->device copies of the e2e step ran at half speed).  Best effort; returns the CPU list
    or None."""
    try:
        import pynvml

        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(index)
        n = os.cpu_count() or 64
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (n + 63) // 64)
        cpus = [w * 64 + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1 and w * 64 + b < n]
        avail = os.sched_getaffinity(0)
        cpus = [c for c in cpus if c in avail]
        if cpus:
            os.sched_setaffinity(0, cpus)
            return cpus
    except Exception:
        pass
    return None


def _barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def _max_over_ranks(v: float, world: int, dev) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist

    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _sum_over_ranks(v: float, world: int, dev) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist

    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def time_workload(wl, steps: int, warmup: int, world: int, dev, split_every: int = 4, sampler=None):
    """W untimed warm-up steps, then K timed steps bracketed by barrier + synchronize, CUDA events on
    the launching stream.  Returns ms per step (block time / K, max over ranks), the per-step times
    (min / median, per-step events), the live per-segment split and the library launches."""
    import torch

    import paper_2001_00706_b200 as sb

    stream = wl.stream
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    flush = torch.empty(256 * 2 ** 20 // 4, dtype=torch.float32, device=dev) if wl.flush else None
    for _ in range(warmup):
        wl.step()
    torch.cuda.synchronize(dev)
    graph = None
    if wl.graph:
        # latency-bound step (c1: ~10 us of GPU work behind ~20 us of Python launch overhead): the
        # step's C-ABI calls are captured once in a CUDA graph and replayed -- the same kernels on
        # the same inputs every step, without the host launch cost between them
        side = torch.cuda.Stream(dev)
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            wl.step()
        stream.wait_stream(side)
        graph = torch.cuda.CUDAGraph()
        c0 = sb.lib().sig_launch_count()
        with torch.cuda.graph(graph):
            wl.step()
        graph_launches = sb.lib().sig_launch_count() - c0  # kernels per replayed step
        torch.cuda.synchronize(dev)
        split_every = 0
    _barrier(world)
    torch.cuda.synchronize(dev)
    launches0 = sb.lib().sig_launch_count()
    marks, splits = [], []
    import contextlib

    with (sampler if sampler is not None else contextlib.nullcontext()):
        t_start, t_end = ev(), ev()
        t_start.record(stream)
        for i in range(steps):
            if flush is not None:
                flush.zero_()  # evict the previous step's data from L2 (outside the per-step events)
            a, b = ev(), ev()
            a.record(stream)
            if graph is not None:
                graph.replay()
            elif split_every and i % split_every == 0:
                rec = []
                wl.step(rec)
                splits.append(rec)
            else:
                wl.step()
            b.record(stream)
            marks.append((a, b))
        t_end.record(stream)
        torch.cuda.synchronize(dev)
    _barrier(world)
    torch.cuda.synchronize(dev)
    launches = sb.lib().sig_launch_count() - launches0
    if graph is not None:
        launches = graph_launches * steps
    per_step = [a.elapsed_time(b) for a, b in marks]
    # with flushes between steps the block time includes them: the step time is the sum of the steps
    block = sum(per_step) if flush is not None else t_start.elapsed_time(t_end)
    ms_step = _max_over_ranks(block, world, dev) / steps
    seg = {}
    for rec in splits:
        for (la, ea), (lb, eb) in zip(rec, rec[1:]):
            seg.setdefault(lb, []).append(ea.elapsed_time(eb))
    seg_ms = {k: float(np.mean(v)) for k, v in seg.items()}
    if graph is not None:
        seg_ms = {"fwd": float(np.mean(per_step))}  # one forward launch per step
    return {"ms_step": ms_step, "graph": graph is not None, "ms_min": _max_over_ranks(float(np.min(per_step)), world, dev),
            "ms_median": _max_over_ranks(float(np.median(per_step)), world, dev), "seg_ms": seg_ms,
            "launches": int(launches)}


def measure_e2e(wl, steps: int, world: int, dev):
    """The same step through the C ABI from pinned host buffers (H2D inputs, D2H result, every step)."""
    import torch

    stream = wl.stream
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    wl.prepare_e2e()
    n_e2e = max(3, min(steps, 50))
    for _ in range(10):  # the first passes over fresh pinned buffers run slow
        wl.e2e_step()
    torch.cuda.synchronize(dev)
    _barrier(world)
    a, b = ev(), ev()
    a.record(stream)
    for _ in range(n_e2e):
        wl.e2e_step()
    b.record(stream)
    torch.cuda.synchronize(dev)
    e_ms = _max_over_ranks(a.elapsed_time(b) / n_e2e, world, dev)
    # context for the e2e number: the plain pinned H2D bandwidth of this box, same buffers (it varied
    # 37-55 GB/s between boxes and runs during development)
    src = wl.gh if wl.gh is not None else wl.xh
    dst = torch.empty(src.shape, dtype=src.dtype, device=dev)
    dst.copy_(src, non_blocking=True)
    a.record(stream)
    for _ in range(3):
        dst.copy_(src, non_blocking=True)
    b.record(stream)
    torch.cuda.synchronize(dev)
    h2d_gbs = 3 * src.numel() * 4 / (a.elapsed_time(b) / 1000) / 1e9
    del dst
    units = _sum_over_ranks(wl.units, world, dev)
    return {"value": units / (e_ms / 1000), "unit": UNIT,
            "h2d_bytes_per_step": int(wl.h2d), "d2h_bytes_per_step": int(wl.d2h),
            "h2d_gbs_probe": round(h2d_gbs, 1),
            "path": ("C ABI calls from pinned host buffers (inputs H2D, result D2H inside the timed region)" +
                     ("; sig_signature_fwd_bwd_host: one C-ABI call on the host buffers, 4 batch slices whose "
                      "copies overlap the kernels" if wl.pipe is not None else ""))}


def measure_e2e_train(wl, steps: int, world: int, dev):
    """The fwd + bwd step as a training step through the public autograd API: per step the batch of
    paths goes host -> device (pinned), out = signature(x), loss = <W, out> with W [S] a
    device-resident linear head, loss.backward() (the reversible backward kernels), and the loss
    comes back device -> host.  The upstream gradient is produced on the device, as in training;
    `e2e` (above) is the stricter variant that also ships a [B, S] upstream gradient from the host."""
    import torch

    sb, N = wl.sb, wl.N
    stream = wl.stream
    xh = torch.from_numpy(wl.x_np).pin_memory()
    xd = [torch.empty(xh.shape, dtype=torch.float32, device=dev) for _ in range(2)]
    W = torch.from_numpy(normal((wl.S,), 4242)).to(dev)
    lossh = torch.empty((), dtype=torch.float32).pin_memory()
    # a data loader's double buffering: the next batch's H2D runs on a copy stream while this batch
    # computes (every batch is still copied inside the timed region)
    cstream = torch.cuda.Stream(dev)
    arrived = [torch.cuda.Event(), torch.cuda.Event()]
    consumed = [torch.cuda.Event(), torch.cuda.Event()]
    it = [0]

    def load(k):
        with torch.cuda.stream(cstream):
            cstream.wait_event(consumed[k])
            xd[k].copy_(xh, non_blocking=True)
            arrived[k].record(cstream)

    def step():
        k = it[0] % 2
        load(1 - k)  # the next batch
        stream.wait_event(arrived[k])
        x = xd[k].detach().requires_grad_(True)
        loss = (sb.signature(x, N) @ W).sum()
        loss.backward()
        consumed[k].record(stream)
        lossh.copy_(loss.detach(), non_blocking=True)
        it[0] += 1

    for ev_ in consumed:
        ev_.record(stream)
    load(0)

    for _ in range(5):
        step()
    torch.cuda.synchronize(dev)
    _barrier(world)
    n = max(3, min(steps, 50))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(n):
        step()
    b.record(stream)
    torch.cuda.synchronize(dev)
    e_ms = _max_over_ranks(a.elapsed_time(b) / n, world, dev)
    units = _sum_over_ranks(wl.units, world, dev)
    return {"value": units / (e_ms / 1000), "unit": UNIT, "h2d_bytes_per_step": int(xh.numel() * 4),
            "d2h_bytes_per_step": 4,
            "path": "autograd: signature(x) -> loss = <W, Sig> (W [S] on the device) -> loss.backward(); "
                    "paths H2D (double-buffered on a copy stream) and the loss D2H every step"}


def _metric_name(name):
    return METRIC if name == "c2" else f"{CONFIGS[name]['op']} paths/sec ({name})"


def measure_config(name, rank, world, dev, steps, warmup, scaling="weak", batch=None):
    """A bounded measurement of one BASELINE config (the `configs` block and the strong/weak arm)."""
    wl = Workload(name, rank, world, dev, scaling=scaling, batch=batch)
    r = time_workload(wl, steps, warmup, world, dev)
    units = _sum_over_ranks(wl.units, world, dev)
    out = {"metric": _metric_name(name), "value": units / (r["ms_step"] / 1000), "unit": UNIT,
           "ms_per_step": r["ms_step"], "ms_min": r["ms_min"], "ms_median": r["ms_median"], "steps": steps,
           "warmup": warmup, "scaling": wl.scaling,
           "config": _config_dict(name, world, wl.scaling, wl.B_global if wl.scaling == "strong" else wl.B, wl.l2),
           "roofline": wl.roofline(r["seg_ms"], r["ms_step"]), "gpu_launches": r["launches"],
           "cuda_graph": r["graph"]}
    del wl
    return out


def run_ours(args, rank: int, world: int):
    import torch

    dev = torch.device("cuda", _local_gpu())
    all_cpus = os.sched_getaffinity(0)
    bind_gpu_local_cpus(dev.index)
    torch.cuda.set_device(dev)
    wl = Workload(args.config, rank, world, dev, scaling=args.scaling, batch=args.batch)
    sampler = ClockSampler(dev.index)
    r = time_workload(wl, args.steps, args.warmup, world, dev, sampler=sampler)
    ms_step = r["ms_step"]
    units = _sum_over_ranks(wl.units, world, dev)
    value = units / (ms_step / 1000.0)
    roofline = wl.roofline(r["seg_ms"], ms_step)
    e2e = measure_e2e(wl, args.steps, world, dev)
    e2e_train = measure_e2e_train(wl, args.steps, world, dev) if wl.cfg["op"] == "sig_fwd_bwd" else None
    scaling = wl.scaling
    line = {
        "metric": _metric_name(args.config),
        "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "ms_min": r["ms_min"], "ms_median": r["ms_median"],
        "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": _config_dict(args.config, world, scaling, wl.B_global if scaling == "strong" else wl.B, wl.l2),
        "roofline": roofline, "e2e": e2e, "clocks": sampler.summary(), "gpu_launches": r["launches"],
    }
    if e2e_train is not None:
        line["e2e_train"] = e2e_train
    del wl
    torch.cuda.empty_cache()
    # the other scaling mode of a batch-sharded config, measured in the same run (at N = 1 both
    # modes are the same workload)
    if world > 1 and args.config in ("c2", "c4") and not args.no_configs:
        other = "strong" if scaling == "weak" else "weak"
        line[other] = measure_config(args.config, rank, world, dev, min(args.steps, 100), args.warmup,
                                     scaling=other, batch=args.batch)
    # every other BASELINE config, bounded, in the same run (c1 is a single-GPU row)
    if not args.no_configs:
        blk = {}
        for name in ("c1", "c2", "c3", "c4", "c5", "c5b", "c3l"):
            if name == args.config or (name == "c1" and world > 1):
                continue
            blk[name] = measure_config(name, rank, world, dev, min(args.steps, 50), args.warmup)
            torch.cuda.empty_cache()
        line["configs"] = blk
    if rank != 0:
        return
    if world == 1 and not args.no_cpu_baseline:
        os.sched_setaffinity(0, all_cpus)  # the oracle gets every host core, not just the GPU-local ones
        line["cpu_baseline"] = cpu_baseline(args.config, seconds=args.cpu_seconds)
    print(json.dumps(line), flush=True)


def run_dry(args, rank: int, world: int):
    """--dry-run: the launch / rendezvous / timing / max-over-ranks / JSON path on CPU (gloo), no
    kernels and no oracle -- for the CPU tests of the multi-process bench."""
    import torch

    x = torch.randn(64, 64)
    ts = []
    for _ in range(args.warmup):
        x = torch.tanh(x @ x.T / 64)
    _barrier(world)
    for _ in range(args.steps):
        t0 = time.perf_counter()
        x = torch.tanh(x @ x.T / 64)
        ts.append((time.perf_counter() - t0) * 1000)
    _barrier(world)
    ms = _max_over_ranks(float(np.sum(ts)), world, torch.device("cpu")) / args.steps
    if rank == 0:
        print(json.dumps({"metric": _metric_name(args.config), "dry_run": True, "n_gpus": world,
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                          "backend": args.backend, "scaling": args.scaling}), flush=True)


def _local_gpu() -> int:
    """This rank's GPU: LOCAL_RANK.  Dev check only: SIGB200_BENCH_SHARE_GPU=1 puts every rank on
    cuda:0 (with --backend gloo) to exercise the N-rank path of this script on a one-GPU box; the
    numbers of such a run are not a measurement of N GPUs."""
    if os.environ.get("SIGB200_BENCH_SHARE_GPU") == "1":
        return 0
    return int(os.environ.get("LOCAL_RANK", 0))


def _free_port() -> int:
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=None, help="ranks (one per GPU); launches them itself if needed")
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="c2")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak",
                    help="batch-sharded configs: weak = B paths per GPU, strong = B paths over all GPUs")
    ap.add_argument("--batch", type=int, default=None, help="override the config's batch B (per-shard studies)")
    ap.add_argument("--backend", choices=["nccl", "gloo"], default=None)
    ap.add_argument("--dry-run", action="store_true", help="CPU orchestration check: no kernels, no oracle")
    ap.add_argument("--no-configs", action="store_true", help="skip the other configs / the other scaling arm")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    env_world = os.environ.get("WORLD_SIZE")
    gpus = args.gpus if args.gpus is not None else (int(env_world) if env_world else 1)
    if env_world is None and gpus > 1:
        # one process per GPU: re-launch this script under torchrun (rendezvous on 127.0.0.1)
        import subprocess

        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)]
        cmd += sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    world = int(env_world or "1")
    if args.gpus is not None and args.gpus != world:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: refusing to measure a different world size")
    rank = int(os.environ.get("RANK", "0"))
    args.backend = args.backend or ("gloo" if args.dry_run else "nccl")
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        if not args.dry_run:
            torch.cuda.set_device(_local_gpu())
        dist.init_process_group(args.backend)
    try:
        (run_dry if args.dry_run else run_ours)(args, rank, world)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
