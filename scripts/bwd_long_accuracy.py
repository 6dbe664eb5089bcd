"""Dev: reversible backward accuracy vs the float64 oracle for long paths, chunked (small B) and not."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle
import paper_2001_00706_b200 as sb
from synth import brownian_paths, normal
from tests.parity import path_rel_err

C, N = 3, 6
for B, L in [(20, 20001), (150, 20001), (1, 200001)]:
    x = brownian_paths(B, L, C, seed=5)
    g = normal((B, oracle.sig_channels(C, N)), seed=105)
    xt = torch.from_numpy(x).cuda()
    gp, _ = sb.sig_signature_backward(torch.from_numpy(g).cuda(), xt, sb.sig_signature(xt, N), N)
    ref, _ = oracle.signature_vjp(g, x, N, threads=16)
    print(f"B={B} L={L}: {path_rel_err(gp.cpu().numpy(), ref):.3e}", flush=True)
