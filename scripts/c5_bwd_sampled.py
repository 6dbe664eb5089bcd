"""Dev: sampled float64 check of the c5-shaped backward (256 oracle chunks, gradient of 3 chunks)
for the libraries in argv[2:] at L = argv[1]."""
import os, subprocess, sys
L = int(sys.argv[1])
code = r'''
import sys, numpy as np, torch
from concurrent.futures import ThreadPoolExecutor
sys.path.insert(0, ".")
import oracle
import paper_2001_00706_b200 as sb
from synth import brownian_paths, normal
from tests.parity import path_rel_err
C, N, L = 3, 6, %d
x = brownian_paths(1, L, C, seed=5)
g = normal((1, oracle.sig_channels(C, N)), seed=105)
xt = torch.from_numpy(x).cuda()
gp, _ = sb.sig_signature_backward(torch.from_numpy(g).cuda(), xt, sb.sig_signature(xt, N), N)
gp = gp.cpu().numpy()
np.save("/tmp/gp_%%s.npy" %% sys.argv[1], gp)
nch, M = 256, L - 1
e = [round(j * M / nch) for j in range(nch + 1)]
with ThreadPoolExecutor(16) as ex:
    sigs = np.stack(list(ex.map(lambda j: oracle.signature(x[:, e[j]:e[j + 1] + 1], N)[0], range(nch))))
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
    print(j, "err", path_rel_err(gp[:, a:b], ref[:, 1:-1]), "max|ref|", np.abs(ref).max(), flush=True)
''' % L
for lib in sys.argv[2:]:
    env = dict(os.environ, SIGB200_LIB=os.path.abspath(lib))
    out = subprocess.run([sys.executable, "-c", code, os.path.basename(lib)], env=env, capture_output=True, text=True)
    print(os.path.basename(lib), L, out.stdout.strip(), out.stderr.strip()[-500:], flush=True)
