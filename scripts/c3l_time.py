"""Dev: stream-mode logsignature (words) at c3's shape, time per call, for the libraries in argv."""
import os, subprocess, sys
code = r'''
import sys, torch
sys.path.insert(0, ".")
import paper_2001_00706_b200 as sb
from synth import brownian_paths
x = torch.from_numpy(brownian_paths(256, 1024, 6, 3)).cuda()
for _ in range(3): sb.sig_logsignature(x, 4, "words", stream=True)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20): sb.sig_logsignature(x, 4, "words", stream=True)
e.record(); torch.cuda.synchronize()
print(round(s.elapsed_time(e) / 20 * 1000, 1), "us/call")
'''
for lib in sys.argv[1:]:
    env = dict(os.environ, SIGB200_LIB=os.path.abspath(lib))
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(os.path.basename(lib), out.stdout.strip(), out.stderr.strip()[-400:])
