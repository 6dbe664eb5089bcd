"""Dev/profiling driver: a few c2 fwd+bwd steps (for ncu launch lists and --set full captures)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2001_00706_b200 as sb
from synth import brownian_paths, normal, CONFIGS

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
c = CONFIGS[cfg if cfg in CONFIGS else "c5"]
x = torch.from_numpy(brownian_paths(c["B"], c["L"], c["C"], 2)).cuda()
if cfg == "c2":
    g = torch.from_numpy(normal((c["B"], sb.sig_signature_channels(c["C"], c["N"])), 102)).cuda()
    for _ in range(steps):
        out = sb.sig_signature(x, c["N"])
        sb.sig_signature_backward(g, x, out, c["N"])
elif cfg == "c4":
    g = torch.from_numpy(normal((c["B"], 3304), 104)).cuda()
    for _ in range(steps):
        o, s = sb.sig_logsignature(x, c["N"], "words", return_signature=True)
        sb.sig_logsignature_backward(g, x, s, c["N"], "words")
elif cfg == "c5b":
    c = CONFIGS["c5"]
    x = torch.from_numpy(brownian_paths(c["B"], c["L"], c["C"], 5)).cuda()
    g = torch.from_numpy(normal((c["B"], sb.sig_signature_channels(c["C"], c["N"])), 105)).cuda()
    for _ in range(steps):
        out = sb.sig_signature(x, c["N"])
        sb.sig_signature_backward(g, x, out, c["N"])
else:
    for _ in range(steps):
        sb.sig_signature(x, c["N"], stream=c["stream"])
torch.cuda.synchronize()
print("ok")
