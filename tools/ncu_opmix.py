"""Per-opcode executed-instruction mix of an ncu report (SASS source page),
per unit of work.  Usage: python tools/ncu_opmix.py rep units [top]"""
import collections
import csv
import io
import subprocess
import sys

rep, units = sys.argv[1], int(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ix = {k: i for i, k in enumerate(h)}
mix = collections.Counter()
for r in rows[2:]:
    c = int(r[ix["Instructions Executed"]] or 0)
    toks = r[ix["Source"]].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
    mix[op.split(".")[0]] += c
tot = sum(mix.values())
print(f"total {tot / units:.1f} warp-instructions per unit")
for op, c in mix.most_common(top):
    print(f"{op:12s} {c / units:10.1f}  {100 * c / tot:5.1f}%")
