"""Dev: small calls of every kernel family, for compute-sanitizer (memcheck / racecheck / synccheck)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2001_00706_b200 as sb
from synth import brownian_paths, normal

def cu(a):
    return torch.from_numpy(a).cuda()

# two-prefix forward/backward (C=8, N=4, B >= 148), basepoint given
x = cu(brownian_paths(150, 9, 8, 1))
bp = cu(normal((150, 8), 2))
s = sb.sig_signature(x, 4, basepoint=bp)
g = cu(normal((150, s.shape[1]), 3))
sb.sig_signature_backward(g, x, s, 4, basepoint=bp)
# one-prefix kernels, stream mode (staged TMA rows, odd S, several paths per CTA)
x2 = cu(brownian_paths(400, 13, 5, 4))
st = sb.sig_signature(x2, 3, stream=True)
sb.sig_signature_backward(cu(normal(tuple(st.shape), 5)), x2, st, 3, stream=True)
# time-chunked long path, forward and backward
x3 = cu(brownian_paths(1, 5000, 3, 6))
s3 = sb.sig_signature(x3, 4)
sb.sig_signature_backward(cu(normal((1, s3.shape[1]), 7)), x3, s3, 4)
# logsignature (compiled K4/K5) words and brackets
x4 = cu(brownian_paths(3, 20, 4, 8))
for mode in ("words", "brackets", "expand"):
    o, sg = sb.sig_logsignature(x4, 5, mode, return_signature=True)
    sb.sig_logsignature_backward(cu(normal(tuple(o.shape), 9)), x4, sg, 5, mode)
# round 2: prefix-pair K2 (c2's shape), latency plan with the register fold (c1's shape), one-warp
# chunked K2 with per-tile staging and the compiled blocked scans (C=3, N=6), plain unchunked long
# backward (C API without workspace)
x5 = cu(brownian_paths(150, 12, 8, 10))
s5 = sb.sig_signature(x5, 5)
sb.sig_signature_backward(cu(normal((150, s5.shape[1]), 11)), x5, s5, 5)
x6 = cu(brownian_paths(4, 128, 4, 12))
sb.sig_signature(x6, 4)
x7 = cu(brownian_paths(1, 20000, 3, 13))
s7 = sb.sig_signature(x7, 6)
sb.sig_signature_backward(cu(normal((1, s7.shape[1]), 14)), x7, s7, 6)
g7 = cu(normal((1, s7.shape[1]), 15))
gp7 = torch.empty_like(x7)
Lib = sb.lib()
assert Lib.sig_signature_backward(sb._ptr(g7), sb._ptr(x7), sb._ptr(s7), 1, 20000, 3, 6, 0, sb.BP_NONE, None,
                                  sb._ptr(gp7), None, sb._stream(x7.device)) == 0
# round 2: forward with saved chunk states and the backward that starts from them
o8, sv8 = sb.sig_signature_save(x7, 6)
sb.sig_signature_backward_saved(g7, x7, o8, sv8, 6)
torch.cuda.synchronize()
print("ok")
