"""Dev: c4 step (logsignature words fwd + bwd, B=512 L=256 C=4 N=7) and its backward alone, per
call, for the libraries in argv."""
import os, subprocess, sys
code = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2001_00706_b200 as sb
from synth import brownian_paths, normal
x = torch.from_numpy(brownian_paths(512, 256, 4, 4)).cuda()
g = torch.from_numpy(normal((512, sb.sig_logsignature_channels(4, 7, "words")), 104)).cuda()
o, s = sb.sig_logsignature(x, 7, "words", return_signature=True)
def t(f, n=30):
    for _ in range(3): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1000
step = t(lambda: sb.sig_logsignature_backward(g, x, sb.sig_logsignature(x, 7, "words", return_signature=True)[1], 7, "words"))
bwd = t(lambda: sb.sig_logsignature_backward(g, x, s, 7, "words"))
sb2 = t(lambda: sb.sig_signature_backward(torch.ones_like(s), x, s, 7))
print(f"step {step:.1f} us, logsig bwd {bwd:.1f} us, sig bwd {sb2:.1f} us")
'''
for lib in sys.argv[1:]:
    env = dict(os.environ, SIGB200_LIB=os.path.abspath(lib))
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(os.path.basename(lib), out.stdout.strip(), out.stderr.strip()[-400:])
