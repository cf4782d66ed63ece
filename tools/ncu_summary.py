"""Summarise an ncu report: key SOL metrics, per-instruction-class counts and
stall reasons (from the SASS source page).  Usage: python tools/ncu_summary.py rep [M]"""
import csv
import collections
import io
import subprocess
import sys

rep = sys.argv[1]
M = int(sys.argv[2]) if len(sys.argv) > 2 else 0


def run(args):
    return subprocess.run(["ncu", "-i", rep] + args, capture_output=True, text=True).stdout


det = list(csv.reader(io.StringIO(run(["--page", "details", "--csv"]))))
hdr = det[0]
want = ["Duration", "Elapsed Cycles", "SM Frequency", "Executed Ipc Active", "Issue Slots Busy", "Compute (SM) Throughput",
        "Memory Throughput", "DRAM Throughput", "L2 Cache Throughput", "Registers Per Thread", "Achieved Active Warps Per SM",
        "Eligible Warps Per Scheduler", "No Eligible", "Executed Instructions", "Warp Cycles Per Issued Instruction"]
for row in det[1:]:
    d = dict(zip(hdr, row))
    if d.get("Metric Name") in want:
        print(f"{d['Metric Name']:40s} {d['Metric Value']:>16s} {d.get('Metric Unit','')}")
raw = list(csv.reader(io.StringIO(run(["--page", "raw", "--csv"]))))
rh = raw[0]
vals = dict(zip(rh, raw[2])) if len(raw) > 2 else {}
for k in ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
          "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
          "smsp__issue_active.avg.pct_of_peak_sustained_active"]:
    for kk in rh:
        if kk.startswith(k):
            print(f"{kk:75s} {vals.get(kk,'')}")
src = list(csv.reader(io.StringIO(run(["--page", "source", "--csv", "--print-source", "sass"]))))
h = src[1]
ix = {k: i for i, k in enumerate(h)}
stall_cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = collections.Counter()
for r in src[2:]:
    for c in stall_cols:
        try:
            tot[c] += int(r[ix[c]] or 0)
        except ValueError:
            pass
s = sum(tot.values()) or 1
print("stall reasons (all samples):", ", ".join(f"{k[6:]} {v / s:.1%}" for k, v in tot.most_common(8)))
if M:
    cls = collections.Counter()
    for r in src[2:]:
        cls[int(r[ix["Instructions Executed"]] or 0)] += 1
    tot_i = sum(c * k for c, k in cls.items())
    print(f"warp-instructions per candidate: {tot_i / M:.1f}")
    for c, k in sorted(cls.items(), key=lambda x: -x[0] * x[1])[:12]:
        print(f"  {c:>12} x {k:>4} = {c * k / M:8.1f} per candidate")
    if len(sys.argv) > 3:
        # the hottest SASS lines (executions per candidate) with their text
        rows = sorted(src[2:], key=lambda r: -int(r[ix["Instructions Executed"]] or 0))[: int(sys.argv[3])]
        for r in rows:
            c = int(r[ix["Instructions Executed"]] or 0)
            print(f"  {c / M:8.2f}  {r[ix['Address']]:>6s}  {r[ix['Source']][:80]}")
