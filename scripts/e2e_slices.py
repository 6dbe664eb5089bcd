"""Dev: c2 end-to-end through the native host entry point (sig_signature_fwd_bwd_host) with 2..16
batch slices, GPU-local CPUs bound, one process."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2001_00706_b200 as sb
from bench import bind_gpu_local_cpus
from synth import brownian_paths, normal

bind_gpu_local_cpus(0)
x = torch.from_numpy(brownian_paths(1024, 128, 8, 2)).pin_memory()
g = torch.from_numpy(normal((1024, 37448), 102)).pin_memory()
out = torch.empty((1024, 128, 8)).pin_memory()
for chunks in (2, 4, 6, 8, 12, 16):
    f = lambda: sb.sig_signature_fwd_bwd_host(x, g, 5, chunks=chunks, grad_path_h=out)
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20):
        f()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 20
    print(f"chunks {chunks}: {ms:.3f} ms/step, {1024 / ms * 1000:.0f} paths/s")
