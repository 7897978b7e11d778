#!/usr/bin/env python3
"""Top SASS instructions of an ncu report by one stall reason, with the CUDA
source line they map to (ncu -i R --page source --csv --print-source cuda,sass).

  ncu_stalls.py REPORT [stall_column=stall_wait] [top=30]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
col = sys.argv[2] if len(sys.argv) > 2 else "stall_wait"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
hdr, out, fname = None, [], "?"
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0].isdigit() and len(r) == len(hdr):
        try:
            v = float(r[hdr.index(col)])
        except (ValueError, IndexError):
            continue
        out.append((v, f"{fname}:{r[0]}", r[1][:70], r[3][:60]))
tot = sum(x[0] for x in out) or 1
print(col, "total", tot)
for v, loc, src, sass in sorted(out, reverse=True)[:top]:
    print(f"{100 * v / tot:5.1f}% {loc:28s} {sass:60s} | {src}")
