"""Turn gpurun_out ncu artefacts into the committed text summaries under
profiles/ (per-kernel share of the bench step, top-kernel ncu summary,
DRAM traffic per launch for bench.py's roofline.traffic).

    python tools/make_profiles.py <round> <launches.csv> <top.ncu-rep> <cands_in_top> [traffic.ncu-rep cands]"""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rnd, launches, top, cands = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4])
out = os.path.join(ROOT, "profiles")
os.makedirs(out, exist_ok=True)

rows = [r for r in csv.reader(open(launches)) if len(r) > 5]
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in rows[1:]:
    if r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    v = float(r[ix["Metric Value"]].replace(",", ""))
    v *= {"ms": 1e6, "us": 1e3, "ns": 1.0, "s": 1e9}.get(r[ix["Metric Unit"]], 1.0)
    name = r[ix["Kernel Name"]].split("(")[0]
    tot[name] += v
    cnt[name] += 1
s = sum(tot.values())
with open(os.path.join(out, f"{rnd}_launch_shares.txt"), "w") as f:
    f.write("# ncu --metrics gpu__time_duration.sum --clock-control none, one bench.py step (+warm-up):\n")
    f.write("# cold-cache serialised launches; compare SHARES, not absolute times\n")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        f.write(f"{v / 1e6:12.3f} ms  {100 * v / s:6.2f}%  x{cnt[k]:3d}  {k}\n")
subprocess.run(["cp", launches, os.path.join(out, f"{rnd}_launches.csv")])
summ = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), top, str(cands)],
                      capture_output=True, text=True).stdout
with open(os.path.join(out, f"{rnd}_k_mc_stats_mma_ncu_summary.txt"), "w") as f:
    f.write(f"# ncu --set full --clock-control none, k_mc_stats_mma, C2 shape, {cands} candidates per launch\n")
    f.write(summ)
if len(sys.argv) > 6:
    trep, tc = sys.argv[5], int(sys.argv[6])
    raw = list(csv.reader(subprocess.run(["ncu", "-i", trep, "--page", "raw", "--csv"], capture_output=True,
                                         text=True).stdout.splitlines()))
    h = raw[0]
    unit = dict(zip(h, raw[1]))
    vals = dict(zip(h, raw[2]))

    def bytes_of(k):
        v = float(vals[k].replace(",", ""))
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit[k], 1)

    b = bytes_of("dram__bytes_read.sum") + bytes_of("dram__bytes_write.sum")
    json.dump({"k_mc_stats_mma_bytes_per_launch": b, "candidates_per_launch": tc,
               "bytes_per_candidate": b / tc, "algorithmic_bytes_per_candidate": 8,
               "source": os.path.basename(trep)}, open(os.path.join(out, "traffic.json"), "w"), indent=1)
print(open(os.path.join(out, f"{rnd}_launch_shares.txt")).read())
print(summ)
