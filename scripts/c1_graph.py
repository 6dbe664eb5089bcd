"""Dev: c1 forward per call, eager vs replayed from a CUDA graph, for the libraries in argv."""
import os, subprocess, sys
code = r'''
import sys, torch
sys.path.insert(0, ".")
import paper_2001_00706_b200 as sb
from synth import brownian_paths
x = torch.from_numpy(brownian_paths(32, 128, 4, 1)).cuda()
def t(f, n=400):
    for _ in range(20): f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n): f()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / n * 1000
eager = t(lambda: sb.sig_signature(x, 4))
st = torch.cuda.Stream()
st.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(st):
    for _ in range(3): sb.sig_signature(x, 4)
torch.cuda.current_stream().wait_stream(st)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    out = sb.sig_signature(x, 4)
graph = t(lambda: g.replay())
print(f"eager {eager:.2f} us/call, graph replay {graph:.2f} us/call")
'''
for lib in sys.argv[1:]:
    env = dict(os.environ, SIGB200_LIB=os.path.abspath(lib))
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(os.path.basename(lib), out.stdout.strip(), out.stderr.strip()[-500:])
