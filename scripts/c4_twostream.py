"""Dev: c4 step as one call vs the batch split in two halves on two CUDA streams (do the halves'
partial last waves overlap?)."""
import sys, torch
sys.path.insert(0, ".")
import paper_2001_00706_b200 as sb
from synth import brownian_paths, normal
x = torch.from_numpy(brownian_paths(512, 256, 4, 4)).cuda()
g = torch.from_numpy(normal((512, sb.sig_logsignature_channels(4, 7, "words")), 104)).cuda()
def step(xx, gg):
    o, s = sb.sig_logsignature(xx, 7, "words", return_signature=True)
    return sb.sig_logsignature_backward(gg, xx, s, 7, "words")
main = torch.cuda.current_stream()
ss = [torch.cuda.Stream(), torch.cuda.Stream()]
def split(parts):
    n = len(parts)
    for k, st in enumerate(ss[:n]):
        st.wait_stream(main)
        with torch.cuda.stream(st):
            step(*parts[k])
    for st in ss[:n]:
        main.wait_stream(st)
def t(f, n=30):
    for _ in range(3): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1000
print("one call", round(t(lambda: step(x, g)), 1), "us")
for cut in (256, 296, 148 * 3):
    parts = [(x[:cut].contiguous(), g[:cut].contiguous()), (x[cut:].contiguous(), g[cut:].contiguous())]
    print(f"two streams cut {cut}", round(t(lambda: split(parts)), 1), "us")
