"""Per-SASS-instruction stall breakdown of an ncu report (source page): the top instructions by samples with
their dominant stall reasons, plus kernel-wide totals per reason."""
import csv
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[1]
rows = r[2:]
si = h.index("Warp Stall Sampling (All Samples)")
sc = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
tot = Counter()
for x in rows:
    for i in sc:
        if x[i].isdigit():
            tot[h[i]] += int(x[i])
T = sum(tot.values()) or 1
print("kernel-wide:", ", ".join(f"{k[6:]} {100 * v / T:.1f}%" for k, v in tot.most_common(10)))
idx = sorted(range(len(rows)), key=lambda j: -int(rows[j][si]) if rows[j][si].isdigit() else 0)[:top]
for j in sorted(idx):
    x = rows[j]
    reasons = sorted(((int(x[i]), h[i][6:]) for i in sc if x[i].isdigit() and int(x[i]) > 0), reverse=True)[:3]
    print(f"{j:5d} {int(x[si]):6d}  {x[1][:60]:60s} {reasons}")
