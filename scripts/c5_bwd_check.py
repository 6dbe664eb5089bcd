"""Dev: at L=200001 (C=3, N=6), GPU backward vs (a) the full float64 oracle VJP and (b) the sampled
256-chunk oracle reference, for chunks 0, 137, 255 -- per-chunk normalisation."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle
import paper_2001_00706_b200 as sb
from synth import brownian_paths, normal
from tests.parity import path_rel_err

C, N, L = 3, 6, int(sys.argv[1]) if len(sys.argv) > 1 else 200001
thr = int(sys.argv[2]) if len(sys.argv) > 2 else 1
x = brownian_paths(1, L, C, seed=5)
g = normal((1, oracle.sig_channels(C, N)), seed=105)
xt = torch.from_numpy(x).cuda()
gp, _ = sb.sig_signature_backward(torch.from_numpy(g).cuda(), xt, sb.sig_signature(xt, N), N)
gp = gp.cpu().numpy()
full, _ = oracle.signature_vjp(g, x, N)
print("full-path err", path_rel_err(gp, full), "max|full|", np.abs(full).max(), flush=True)
nch, M = 256, L - 1
e = [round(j * M / nch) for j in range(nch + 1)]
if thr > 1:
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(thr) as ex:
        sigs = np.stack(list(ex.map(lambda j: oracle.signature(x[:, e[j]:e[j + 1] + 1], N)[0], range(nch))))
else:
    sigs = np.stack([oracle.signature(x[:, e[j]:e[j + 1] + 1], N)[0] for j in range(nch)])
for j in (0, 137, nch - 1):
    P = oracle.multi_combine(sigs[:j, None], C, N)[0] if j > 0 else None
    Pn = oracle.multi_combine(sigs[:j + 1, None], C, N)[0]
    if j < nch - 1:
        Q = oracle.multi_combine(sigs[j + 1:, None], C, N)[0]
        gend = oracle.mul_vjp(g[0], Pn, Q, C, N)[0]
    else:
        gend = g[0].astype(np.float64)
    ref, _, _ = oracle.signature_vjp_ex(gend[None], x[:, e[j]:e[j + 1] + 1], N, initial=None if P is None else P[None])
    a, b = e[j] + 1, e[j + 1]
    print(j, "gpu-vs-sampled", path_rel_err(gp[:, a:b], ref[:, 1:-1]), "gpu-vs-full", path_rel_err(gp[:, a:b], full[:, a:b]),
          "sampled-vs-full", path_rel_err(ref[:, 1:-1], full[:, a:b]), flush=True)
