"""Dev/profiling driver: a few c1 forward calls (for ncu)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2001_00706_b200 as sb
from synth import brownian_paths
x = torch.from_numpy(brownian_paths(32, 128, 4, 1)).cuda()
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 5):
    sb.sig_signature(x, 4)
torch.cuda.synchronize()
print("ok")
