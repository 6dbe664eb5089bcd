"""Dev timing helper: CUDA-event timing of the BASELINE configs (not the bench contract)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2001_00706_b200 as sb
from synth import brownian_paths, normal

def t_events(fn, reps=20, warm=3):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        s.record(); fn(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    return min(ts), float(np.median(ts))

def main():
    dev = "cuda"
    # c2
    x = torch.from_numpy(brownian_paths(1024, 128, 8, 2)).to(dev)
    g = torch.from_numpy(normal((1024, 37448), 102)).to(dev)
    out = sb.sig_signature(x, 5)
    print("c2 fwd ms (min, med):", t_events(lambda: sb.sig_signature(x, 5)))
    print("c2 bwd ms (min, med):", t_events(lambda: sb.sig_signature_backward(g, x, out, 5)))
    print("c2 fwd+bwd ms:", t_events(lambda: sb.sig_signature_backward(g, x, sb.sig_signature(x, 5), 5)))
    # c1
    x1 = torch.from_numpy(brownian_paths(32, 128, 4, 1)).to(dev)
    print("c1 fwd ms:", t_events(lambda: sb.sig_signature(x1, 4)))
    # c3
    x3 = torch.from_numpy(brownian_paths(256, 1024, 6, 3)).to(dev)
    print("c3 stream fwd ms:", t_events(lambda: sb.sig_signature(x3, 4, stream=True), reps=10))
    # c4
    x4 = torch.from_numpy(brownian_paths(512, 256, 4, 4)).to(dev)
    g4 = torch.from_numpy(normal((512, 3304), 104)).to(dev)
    def c4():
        o, s = sb.sig_logsignature(x4, 7, "words", return_signature=True)
        sb.sig_logsignature_backward(g4, x4, s, 7, "words")
    print("c4 logsig fwd ms:", t_events(lambda: sb.sig_logsignature(x4, 7, "words")))
    print("c4 fwd+bwd ms:", t_events(c4))
    # c5
    x5 = torch.from_numpy(brownian_paths(1, 2**22, 3, 5)).to(dev)
    print("c5 fwd ms:", t_events(lambda: sb.sig_signature(x5, 6), reps=10))

if __name__ == "__main__" and len(sys.argv) == 1:
    main()


def c5_bwd():
    """c5 path with the time-parallel backward (not a BASELINE metric)."""
    x5 = torch.from_numpy(brownian_paths(1, 2**22, 3, 5)).to("cuda")
    g5 = torch.from_numpy(normal((1, 1092), 105)).to("cuda")
    out = sb.sig_signature(x5, 6)
    print("c5 bwd ms:", t_events(lambda: sb.sig_signature_backward(g5, x5, out, 6), reps=5))


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "c5bwd":
    c5_bwd()
