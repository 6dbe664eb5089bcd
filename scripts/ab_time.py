"""Dev A/B timing: c2 (and optionally c4) fwd / bwd with CUDA events for the libraries named in argv."""
import os, subprocess, sys
libs = sys.argv[1:]
code = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2001_00706_b200 as sb
from synth import brownian_paths, normal
def t(fn, reps=30, warm=5):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        s.record(); fn(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    return round(float(np.median(ts)), 4)
x = torch.from_numpy(brownian_paths(1024, 128, 8, 2)).cuda()
g = torch.from_numpy(normal((1024, 37448), 102)).cuda()
out = sb.sig_signature(x, 5)
r = {"c2_fwd": t(lambda: sb.sig_signature(x, 5)), "c2_bwd": t(lambda: sb.sig_signature_backward(g, x, out, 5))}
x4 = torch.from_numpy(brownian_paths(512, 256, 4, 4)).cuda()
g4 = torch.from_numpy(normal((512, 21844), 104)).cuda()
o4 = sb.sig_signature(x4, 7)
r["c4_sigfwd"] = t(lambda: sb.sig_signature(x4, 7)); r["c4_sigbwd"] = t(lambda: sb.sig_signature_backward(g4, x4, o4, 7))
print(r)
'''
for lib in libs:
    env = dict(os.environ, SIGB200_LIB=os.path.abspath(lib))
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(os.path.basename(lib), out.stdout.strip(), out.stderr.strip()[-300:])
