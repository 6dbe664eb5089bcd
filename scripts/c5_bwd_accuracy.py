"""Dev: accuracy of the reversible backward on long Brownian paths (C=3, N=6) vs the float64 oracle:
relative error of the point gradient dL/dx and of the increment gradient dL/dz (= -cumsum of dL/dx),
normalised by the whole path's max (reading R9)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle
import paper_2001_00706_b200 as sb
from synth import brownian_paths, normal

C, N = 3, 6
for L in [int(a) for a in sys.argv[1:]] or [4097, 32769, 131073]:
    x = brownian_paths(1, L, C, seed=5)
    g = normal((1, oracle.sig_channels(C, N)), seed=105)
    xt = torch.from_numpy(x).cuda()
    gp, _ = sb.sig_signature_backward(torch.from_numpy(g).cuda(), xt, sb.sig_signature(xt, N), N)
    gp = gp.cpu().numpy().astype(np.float64)
    ref, _ = oracle.signature_vjp(g, x, N)
    ex = np.max(np.abs(gp - ref)) / np.max(np.abs(ref))
    gz, rz = -np.cumsum(gp, axis=1)[:, :-1], -np.cumsum(ref, axis=1)[:, :-1]
    ez = np.max(np.abs(gz - rz)) / np.max(np.abs(rz))
    print(f"L={L}: dL/dx rel err {ex:.3e} (max|ref| {np.max(np.abs(ref)):.3e}), dL/dz rel err {ez:.3e} "
          f"(max|ref| {np.max(np.abs(rz)):.3e})", flush=True)
