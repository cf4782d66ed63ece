"""Counters of the bench's dominant kernel at the bench's own size (C2, one
1e8-candidate k_mc_stats_mma launch, captured by ncu) -> profiles/traffic.json
and profiles/issue.json, which bench.py reports as roofline.traffic and
int_roofline.ncu.

    ncu --metrics <METRICS> --clock-control none -k regex:k_mc_stats_mma -s 1 -c 1 \\
        --csv --log-file gpurun_out/r03/bench_kernel.csv python tools/profile_mc.py 100000000
    python tools/bench_kernel_ncu.py gpurun_out/r03/bench_kernel.csv r03"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = ("dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,"
           "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,"
           "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,"
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,"
           "gpu__time_duration.sum")
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "inst": 1, "Kinst": 1e3, "Minst": 1e6, "Ginst": 1e9,
         "%": 0.01, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1}

if __name__ == "__main__":
    path, rnd = sys.argv[1], sys.argv[2]
    cands = int(sys.argv[3]) if len(sys.argv) > 3 else 10**8
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.reader(lines))
    h = rows[0]
    ix = {k: i for i, k in enumerate(h)}
    vals = {}
    for r in rows[1:]:
        unit = r[ix["Metric Unit"]]
        vals[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", "")) * SCALE.get(unit, 1.0)
    src = f"profiles/{rnd}/bench_kernel.csv (ncu, one k_mc_stats_mma launch of {cands} candidates, the bench size)"
    traffic = vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]
    with open(os.path.join(ROOT, "profiles", "traffic.json"), "w") as f:
        json.dump({"k_mc_stats_mma_bytes_per_launch": traffic, "candidates_per_launch": cands,
                   "bytes_per_candidate": traffic / cands, "algorithmic_bytes_per_candidate": 8,
                   "kernel_ms_under_ncu": vals["gpu__time_duration.sum"] * 1e3, "source": src}, f, indent=1)
    with open(os.path.join(ROOT, "profiles", "issue.json"), "w") as f:
        json.dump({"kernel": "k_mc_stats_mma", "source": src,
                   "issue_slots_busy": vals["smsp__issue_active.avg.pct_of_peak_sustained_active"],
                   "pipe_alu": vals["sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"],
                   "pipe_fma": vals["sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"],
                   "pipe_tensor": vals["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"],
                   "warp_instructions_per_candidate": vals["smsp__inst_executed.sum"] / cands}, f, indent=1)
    print(open(os.path.join(ROOT, "profiles", "traffic.json")).read())
    print(open(os.path.join(ROOT, "profiles", "issue.json")).read())
