"""Dev: condense an ncu report (--set full) or a launch-list CSV into a text summary for profiles/."""
import collections
import csv
import subprocess
import sys

KEYS = ("Duration", "SM Frequency", "Elapsed Cycles", "Compute (SM) Throughput", "Memory Throughput",
        "DRAM Throughput", "Executed Ipc Active", "Issue Slots Busy", "No Eligible", "Eligible Warps Per Scheduler",
        "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy", "Dynamic Shared Memory Per Block",
        "Executed Instructions", "L1/TEX Hit Rate", "L2 Hit Rate", "Block Size", "Grid Size", "Waves Per SM")


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    kn, mn, mu, mv = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    seen = set()
    print("kernel:", rows[1][kn])
    for r in rows[1:]:
        if r[mn] in KEYS and r[mn] not in seen:
            seen.add(r[mn])
            print(f"  {r[mn]:36s} {r[mv]:>16s} {r[mu]}")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    hh, uu, vv = rr[0], rr[1], rr[2]
    want = ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum",
            "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum", "smsp__sass_thread_inst_executed_op_fmul_pred_on.sum",
            "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum")
    for name, unit, val in zip(hh, uu, vv):
        if name in want:
            print(f"  {name:60s} {val} {unit}")
    stalls = [(n, v) for n, v in zip(hh, vv) if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued")]
    tot = sum(float(v.replace(",", "") or 0) for _, v in stalls) or 1.0
    top = sorted(stalls, key=lambda nv: -float(nv[1].replace(",", "") or 0))[:6]
    print("  top stall reasons (share of samples):",
          ", ".join(f"{n.replace('smsp__pcsamp_warps_issue_stalled_', '')} {float(v.replace(',', '')) / tot:.0%}" for n, v in top))


def launches(path):
    rows = list(csv.reader(open(path)))
    h = None
    d = collections.defaultdict(list)
    for r in rows:
        if "Kernel Name" in r:
            h = r
            continue
        if h and len(r) == len(h):
            d[r[h.index("Kernel Name")]].append(float(r[h.index("Metric Value")].replace(",", "")))
    tot = sum(sum(v) for v in d.values())
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        print(f"  {k[:70]:70s} n={len(v):4d} mean={sum(v) / len(v) / 1e3:9.1f} us  share={sum(v) / tot:6.1%}")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(f"# {p}")
        (report if p.endswith(".ncu-rep") else launches)(p)
        print()
