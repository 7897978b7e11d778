#!/usr/bin/env python3
"""Warp-stall samples of an ncu report aggregated over source-line regions.

  ncu_regions.py REPORT FILE.cu name:a-b [name:a-b ...]
"""
import csv
import subprocess
import sys

rep, target = sys.argv[1], sys.argv[2]
regions = []
for spec in sys.argv[3:]:
    name, rng = spec.rsplit(":", 1)
    a, b = rng.split("-")
    regions.append((name, int(a), int(b)))
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
hdr, fname, data = None, "?", []
for r in csv.reader(txt.splitlines()):
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0].isdigit() and len(r) > 4:
        try:
            s = float(r[4] or 0)  # Warp Stall Sampling (All Samples)
        except ValueError:
            continue
        data.append((fname, int(r[0]), s))
tot = sum(d[2] for d in data) or 1
for name, a, b in regions:
    s = sum(d[2] for d in data if d[0] == target and a <= d[1] <= b)
    print(f"{name:34s} {100 * s / tot:5.1f}%")
for f in sorted(set(d[0] for d in data) - {target}):
    print(f"{f:34s} {100 * sum(d[2] for d in data if d[0] == f) / tot:5.1f}%")
