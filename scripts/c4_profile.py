"""Dev/profiling driver: a few c4 logsignature (words) fwd + bwd calls (for ncu)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2001_00706_b200 as sb
from synth import brownian_paths, normal
x = torch.from_numpy(brownian_paths(512, 256, 4, 4)).cuda()
g = torch.from_numpy(normal((512, sb.sig_logsignature_channels(4, 7, "words")), 104)).cuda()
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    o, s = sb.sig_logsignature(x, 7, "words", return_signature=True)
    sb.sig_logsignature_backward(g, x, s, 7, "words")
torch.cuda.synchronize()
print("ok")
