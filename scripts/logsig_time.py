"""Dev: c4 K4 (logsignature from a given signature) time for the libraries in argv."""
import os, subprocess, sys
code = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2001_00706_b200 as sb
from synth import brownian_paths
x = torch.from_numpy(brownian_paths(512, 256, 4, 4)).cuda()
sig = sb.sig_signature(x, 7)
f = lambda: sb.signature_to_logsignature(sig, 4, 7, "words")
for _ in range(5): f()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(50): f()
e.record(); torch.cuda.synchronize()
print(round(s.elapsed_time(e) / 50 * 1000, 1), "us/call")
'''
for lib in sys.argv[1:]:
    env = dict(os.environ, SIGB200_LIB=os.path.abspath(lib))
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(os.path.basename(lib), out.stdout.strip(), out.stderr.strip()[-400:])
