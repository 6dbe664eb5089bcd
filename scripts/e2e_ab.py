"""Dev: c2 end-to-end step (pinned host inputs -> kernels -> host result) timed directly and through
hostpipe.HostPipeline with 2/4/8 slices, in one process on one box."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2001_00706_b200 as sb
from paper_2001_00706_b200.hostpipe import HostPipeline
from synth import brownian_paths, normal

if len(sys.argv) > 1 and sys.argv[1] == "bind":
    from bench import bind_gpu_local_cpus
    print("bound to", bind_gpu_local_cpus(0))
B, L, C, N = 1024, 128, 8, 5
x = torch.from_numpy(brownian_paths(B, L, C, 2)).pin_memory()
g = torch.from_numpy(normal((B, 37448), 102)).pin_memory()
out = torch.empty((B, L, C)).pin_memory()
xd, gd = torch.empty_like(x, device="cuda"), torch.empty_like(g, device="cuda")
fn = lambda a, b: sb.sig_signature_backward(b, a, sb.sig_signature(a, N), N)[0]  # noqa: E731


def direct():
    xd.copy_(x, non_blocking=True)
    gd.copy_(g, non_blocking=True)
    out.copy_(fn(xd, gd), non_blocking=True)


def timeit(f, reps=20):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        f()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


t = timeit(direct)
print(f"direct: {t:.3f} ms  {B / t * 1e3:.0f} paths/s  (H2D {157.6 / t:.1f} GB/s equivalent)")
for k in (2, 4, 8):
    p = HostPipeline([x, g], out, chunks=k)
    t = timeit(lambda: p.run(fn))
    print(f"pipeline x{k}: {t:.3f} ms  {B / t * 1e3:.0f} paths/s")
for k in (2, 4, 8):
    t = timeit(lambda: sb.sig_signature_fwd_bwd_host(x, g, N, chunks=k, grad_path_h=out))
    print(f"native x{k}: {t:.3f} ms  {B / t * 1e3:.0f} paths/s")
h = torch.empty(157581312 // 4).pin_memory()
d = torch.empty_like(h, device="cuda")
t = timeit(lambda: d.copy_(h, non_blocking=True))
print(f"H2D alone 157.6 MB: {t:.3f} ms = {157.6 / t:.1f} GB/s")
