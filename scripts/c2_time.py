"""Dev: c2 signature backward alone and the fwd+bwd step (B=1024 L=128 C=8 N=5), per call, for the
libraries in argv."""
import os, subprocess, sys
code = r'''
import sys, torch
sys.path.insert(0, ".")
import paper_2001_00706_b200 as sb
from synth import brownian_paths, normal
x = torch.from_numpy(brownian_paths(1024, 128, 8, 2)).cuda()
s = sb.sig_signature(x, 5)
g = torch.from_numpy(normal(tuple(s.shape), 102)).cuda()
def t(f, n=30):
    for _ in range(3): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1000
bwd = t(lambda: sb.sig_signature_backward(g, x, s, 5))
fwd = t(lambda: sb.sig_signature(x, 5))
print(f"fwd {fwd:.1f} us, bwd {bwd:.1f} us")
'''
for lib in sys.argv[1:]:
    env = dict(os.environ, SIGB200_LIB=os.path.abspath(lib))
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(os.path.basename(lib), out.stdout.strip(), out.stderr.strip()[-400:])
