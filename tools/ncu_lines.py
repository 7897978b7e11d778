#!/usr/bin/env python3
"""Top CUDA source lines by warp-stall samples of an ncu report
(ncu -i R --page source --csv --print-source cuda,sass)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
out, fname = [], "?"
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0].isdigit() and len(r) > 4:
        try:
            s = float(r[4])
        except ValueError:
            continue
        out.append((s, fname, int(r[0]), r[1][:110]))
tot = sum(x[0] for x in out) or 1
print("total samples", tot)
for s, f, l, src in sorted(out, reverse=True)[:top]:
    print(f"{100 * s / tot:5.1f}% {f}:{l}  {src}")
