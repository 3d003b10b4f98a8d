"""Summarise an ncu report's source page: warp-stall samples per CUDA source line (needs -lineinfo)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None
lines = []
fname = ""
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0].isdigit():
        s = int(r[4]) if r[4].isdigit() else 0
        lines.append((s, fname, int(r[0]), r[1]))
tot = sum(x[0] for x in lines) or 1
print(f"total samples {tot}")
for s, f, ln, src in sorted(lines, key=lambda x: -x[0])[:top]:
    print(f"{100*s/tot:5.1f}%  {f}:{ln:<4d} {src.strip()[:100]}")
