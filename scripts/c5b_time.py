"""Dev: c5b pieces (one path, L = 2^22, C = 3, N = 6): the saved-state forward and the backward from
it, per call, for the libraries in argv."""
import os, subprocess, sys
code = r'''
import sys, torch
sys.path.insert(0, ".")
import paper_2001_00706_b200 as sb
from synth import brownian_paths, normal
x = torch.from_numpy(brownian_paths(1, 2 ** 22, 3, 5)).cuda()
g = torch.from_numpy(normal((1, 1092), 6)).cuda()
def t(f, n=10):
    for _ in range(2): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1000
out, sv = sb.sig_signature_save(x, 6)
fwd = t(lambda: sb.sig_signature_save(x, 6))
bwd = t(lambda: sb.sig_signature_backward_saved(g, x, out, sv, 6))
print(f"save-fwd {fwd:.1f} us, bwd-from-saved {bwd:.1f} us")
'''
for lib in sys.argv[1:]:
    env = dict(os.environ, SIGB200_LIB=os.path.abspath(lib))
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(os.path.basename(lib), out.stdout.strip(), out.stderr.strip()[-400:])
