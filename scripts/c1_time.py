"""Dev: c1 forward time per call (back-to-back launches, CUDA events) for the libraries in argv."""
import os, subprocess, sys
code = r'''
import sys, torch
sys.path.insert(0, ".")
import paper_2001_00706_b200 as sb
from synth import brownian_paths
x = torch.from_numpy(brownian_paths(32, 128, 4, 1)).cuda()
for _ in range(20): sb.sig_signature(x, 4)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(400): sb.sig_signature(x, 4)
e.record(); torch.cuda.synchronize()
print(round(s.elapsed_time(e) / 400 * 1000, 2), "us/call")
'''
for lib in sys.argv[1:]:
    env = dict(os.environ, SIGB200_LIB=os.path.abspath(lib))
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(os.path.basename(lib), out.stdout.strip(), out.stderr.strip()[-300:])
