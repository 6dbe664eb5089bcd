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


def fp32_peak_tflops() -> tuple[float, str]:
    """FP32 FMA peak: 148 SMs x 128 FP32 lanes x 2 FLOP x 1.965 GHz (max SM clock in
    MEASURED_PEAKS.json) = 74.45 TFLOP/s.  MEASURED_PEAKS.json carries no FP32 figure; DESIGN.md
    derives this denominator from the guide's unit counts and clocks."""
    mhz = 1965.0
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        mhz = float(mp.get("sm_max_mhz", mhz))
    except Exception:
        pass
    return 148 * 128 * 2 * mhz * 1e6 / 1e12, f"148 SM x 128 lanes x 2 x {mhz:.0f} MHz (derived, DESIGN.md)"


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
    of the same workload (the first paths of the same seeded batch), threads = all cores."""
    import oracle

    cfg = CONFIGS[cfg_name]
    C, N, L = cfg["C"], cfg["N"], cfg["L"]
    cores = os.cpu_count() or 1
    ps, gs = SEEDS[cfg_name]
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
            "sample": f"{n} of {cfg['B']} paths of {cfg_name} (fwd+bwd, float64 C oracle, {min(cores, n)} threads), "
                      f"{dt:.1f} s"}


def _oracle_step(oracle, cfg_name, x, gs, threads):
    cfg = CONFIGS[cfg_name]
    C, N = cfg["C"], cfg["N"]
    S = sum(C ** k for k in range(1, N + 1))
    if cfg["op"] == "sig_fwd_bwd":
        g = normal((x.shape[0], S), gs)
        oracle.signature_vjp(g, x, N, threads=threads)  # includes the forward it needs
    elif cfg["op"] == "logsig_words_fwd_bwd":
        from oracle import lyndon
        g = normal((x.shape[0], lyndon.witt(C, N)), gs)
        oracle.logsignature_vjp(g, x, N, mode="words", threads=threads)
    else:
        oracle.signature(x, N, stream=cfg["stream"], threads=threads)


# ------------------------------------------------------------------------------------------------
def run_reference(args, rank: int, world: int):
    """Reference arm: the float64 oracle, as it stands, on the host cores."""
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    import oracle

    cores = os.cpu_count() or 1
    n = min(cfg["B"], max(cores, 16))
    x = brownian_paths(cfg["B"], cfg["L"], cfg["C"], SEEDS[args.config][0])[:n]
    for _ in range(args.warmup):
        _oracle_step(oracle, args.config, x[:cores], SEEDS[args.config][1], cores)
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
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": min(cores, n), "kind": "oracle",
                         "sample": f"{n} of {cfg['B']} paths per step, float64 C oracle, {min(cores, n)} threads"},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _config_dict(name, world):
    cfg = CONFIGS[name]
    return {"workload": f"{name}: {cfg['op']} B={cfg['B']}/GPU L={cfg['L']} C={cfg['C']} N={cfg['N']}"
                        f"{' stream' if cfg['stream'] else ''}, Brownian",
            "B_per_gpu": cfg["B"], "L": cfg["L"], "C": cfg["C"], "depth": cfg["N"], "stream": cfg["stream"],
            "parallelism": f"batch-shard x{world}" if world > 1 else "single GPU",
            "l2": "per-step working set > 126 MB L2 (grad_out + signature 307 MB); no flush needed"
            if name == "c2" else "see DESIGN.md"}


# ------------------------------------------------------------------------------------------------
def run_ours(args, rank: int, world: int):
    import torch
    import torch.distributed as dist

    import paper_2001_00706_b200 as sb

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    cfg = CONFIGS[args.config]
    assert cfg["op"] == "sig_fwd_bwd", "bench.py times the metric's configuration c2 (see scripts/ for others)"
    B, L, C, N = cfg["B"], cfg["L"], cfg["C"], cfg["N"]
    S = sb.sig_signature_channels(C, N)
    M = L - 1
    ps, gs = SEEDS[args.config]
    x_np = brownian_paths(B, L, C, ps + 7919 * rank)
    g_np = normal((B, S), gs + 7919 * rank)
    x = torch.from_numpy(x_np).to(dev)
    g = torch.from_numpy(g_np).to(dev)
    stream = torch.cuda.current_stream(dev)

    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def step(times=None):
        if times is not None:
            e0, e1, e2 = ev(), ev(), ev()
            e0.record(stream)
        out = sb.sig_signature(x, N)
        if times is not None:
            e1.record(stream)
        gp, _ = sb.sig_signature_backward(g, x, out, N)
        if times is not None:
            e2.record(stream)
            times.append((e0, e1, e2))
        return gp

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    launches0 = sb.lib().sig_launch_count()
    kt = []
    sampler = ClockSampler(dev.index)
    with sampler:
        t_start, t_end = ev(), ev()
        t_start.record(stream)
        for i in range(args.steps):
            step(kt if i % 4 == 0 else None)
        t_end.record(stream)
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    launches = sb.lib().sig_launch_count() - launches0
    ms_total = t_start.elapsed_time(t_end)
    ms_t = torch.tensor([ms_total], device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_step = float(ms_t.item()) / args.steps
    value = world * B / (ms_step / 1000.0)

    fwd_ms = float(np.mean([a.elapsed_time(b) for a, b, _ in kt]))
    bwd_ms = float(np.mean([b.elapsed_time(c) for _, b, c in kt]))
    peak, peak_src = fp32_peak_tflops()
    bwd_flops = alg_flops("bwd", B, M, C, N)
    achieved = bwd_flops / (bwd_ms / 1000) / 1e12
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        traffic = prof.get("c2", {}).get("sig_bwd_kernel")
    except Exception:
        pass
    roofline = {"bound": "alu", "kernel": "sig_bwd_kernel<Shape<8,5,3>> (reversible backward)",
                "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                "peak_source": peak_src, "kernel_ms": bwd_ms, "step_share": bwd_ms / (fwd_ms + bwd_ms),
                "fwd": {"kernel": "sig_fwd_kernel<Shape<8,5,3>>", "kernel_ms": fwd_ms,
                        "achieved": alg_flops("fwd", B, M, C, N) / (fwd_ms / 1000) / 1e12,
                        "frac": alg_flops("fwd", B, M, C, N) / (fwd_ms / 1000) / 1e12 / peak},
                "step_frac": (alg_flops("fwd", B, M, C, N) + bwd_flops) / (ms_step / 1000) / 1e12 / peak}

    # ---- e2e through the C ABI from pinned host buffers
    xh = torch.from_numpy(x_np).pin_memory()
    gh = torch.from_numpy(g_np).pin_memory()
    gph = torch.empty((B, L, C), dtype=torch.float32).pin_memory()
    xd = torch.empty_like(x)
    gd = torch.empty_like(g)

    def e2e_step():
        xd.copy_(xh, non_blocking=True)
        gd.copy_(gh, non_blocking=True)
        out = sb.sig_signature(xd, N)
        gp, _ = sb.sig_signature_backward(gd, xd, out, N)
        gph.copy_(gp, non_blocking=True)

    n_e2e = max(3, min(args.steps, 50))
    for _ in range(3):
        e2e_step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    a, b = ev(), ev()
    a.record(stream)
    for _ in range(n_e2e):
        e2e_step()
    b.record(stream)
    torch.cuda.synchronize(dev)
    e_ms = torch.tensor([a.elapsed_time(b) / n_e2e], device=dev)
    if world > 1:
        dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
    e2e = {"value": world * B / (float(e_ms.item()) / 1000), "unit": UNIT,
           "h2d_bytes_per_step": int(x.numel() * 4 + g.numel() * 4), "d2h_bytes_per_step": int(B * L * C * 4),
           "path": "C ABI (sig_signature + sig_signature_backward) with pinned host buffers"}

    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": _config_dict(args.config, world), "roofline": roofline,
        "e2e": e2e, "clocks": sampler.summary(), "gpu_launches": int(launches),
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.config, seconds=args.cpu_seconds)
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="c2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        dist.init_process_group("nccl")
    try:
        run_ours(args, rank, world)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
