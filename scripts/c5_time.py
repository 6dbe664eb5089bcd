"""Dev: c5 forward (one path, L = 2^22, C = 3, N = 6) time per call for the libraries in argv."""
import os, subprocess, sys
code = r'''
import sys, torch
sys.path.insert(0, ".")
import paper_2001_00706_b200 as sb
from synth import brownian_paths
x = torch.from_numpy(brownian_paths(1, 2 ** 22, 3, 5)).cuda()
for _ in range(5): sb.sig_signature(x, 6)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(30): sb.sig_signature(x, 6)
e.record(); torch.cuda.synchronize()
print(round(s.elapsed_time(e) / 30 * 1000, 1), "us/call")
'''
for lib in sys.argv[1:]:
    env = dict(os.environ, SIGB200_LIB=os.path.abspath(lib))
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(os.path.basename(lib), out.stdout.strip(), out.stderr.strip()[-400:])
