"""Dev check: logsignature backward of every compiled power-of-two (C, N) against the oracle."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2001_00706_b200 as sb
import oracle
from synth import brownian_paths, normal

cases = [(C, N) for C in (1, 2, 4, 8) for N in range(1, 13) if sum(C ** k for k in range(1, N + 1)) <= 6000]
for C, N in cases:
    x = brownian_paths(2, 6, C, seed=C * 31 + N)
    xt = torch.from_numpy(x).cuda().requires_grad_(True)
    for mode in ("expand", "words"):
        y = sb.logsignature(xt, N, mode)
        g = normal(tuple(y.shape), 7)
        (gx,) = torch.autograd.grad(y, xt, torch.from_numpy(g).cuda())
        ref = oracle.logsignature_vjp(g, x, N, mode=mode)
        ref = ref[0] if isinstance(ref, tuple) else ref
        err = np.abs(gx.cpu().numpy() - ref).max() / max(np.abs(ref).max(), 1e-30)
        print(f"C={C} N={N} {mode:6s} rel_err={err:.2e} {'FAIL' if err > 5e-4 else ''}")
