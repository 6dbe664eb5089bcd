"""Dev: per-opcode executed warp instructions and stall samples from an ncu source page (SASS) CSV
(ncu -i R --page source --csv --print-source sass), plus the FP32-pipe FLOP accounting: issued
FLOPs = 2 x (FFMA + 2 FFMA2) + FADD + FMUL + 2 FADD2/FMUL2 thread instructions (FADD/FMUL counted
as one FLOP each), against the algorithmic FLOPs given on the command line."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ia, isrc, ist, ie, ite = (h.index(k) for k in ("Address", "Source", "Warp Stall Sampling (All Samples)",
                                                 "Instructions Executed", "Predicated-On Thread Instructions Executed"))
ops = collections.Counter()
thr = collections.Counter()
stall = collections.Counter()
for r in rows[2:]:
    if len(r) <= ite:
        continue
    s = r[isrc].strip()
    if s.startswith("@"):
        s = s.split(None, 1)[1]
    op = s.split()[0] if s else "?"
    ops[op] += int(r[ie] or 0)
    thr[op] += int(r[ite] or 0)
    stall[op] += int(r[ist] or 0)
tot = sum(ops.values())
ts = sum(stall.values())
print(f"total warp instructions {tot}, stall samples {ts}")
for op, n in ops.most_common(25):
    print(f"  {op:24s} {n:>12d} {100.0 * n / tot:6.2f}%   stall samples {100.0 * stall[op] / max(ts, 1):5.1f}%")
fl = 0
for op, n in thr.items():
    base = op.split(".")[0]
    if base == "FFMA":
        fl += 2 * n
    elif base == "FFMA2":
        fl += 4 * n
    elif base in ("FADD", "FMUL"):
        fl += n
    elif base in ("FADD2", "FMUL2"):
        fl += 2 * n
print(f"issued FP32 FLOPs (FMA = 2) {fl / 1e9:.3f} G")
if len(sys.argv) > 2:
    alg = float(sys.argv[2])
    print(f"algorithmic {alg / 1e9:.3f} G -> issued / algorithmic = {fl / alg:.3f}")
