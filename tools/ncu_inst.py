#!/usr/bin/env python3
"""Top CUDA source lines by warp-level instructions executed in an ncu report
(source page, cuda view): python tools/ncu_inst.py REPORT [TOP] [FILE:A-B=NAME ...]
Optional FILE:A-B=NAME arguments sum the lines A..B of FILE into phase NAME."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
groups = []
for g in sys.argv[3:]:
    fl, rest = g.split(":")
    rng, name = rest.split("=")
    a, b = (int(x) for x in rng.split("-"))
    groups.append((fl, a, b, name))
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
# SASS rows ("", "", address, instruction, ..., Instructions Executed at column 7) are
# attributed to the CUDA line row above them (its own columns may be split by commas)
lines, fname, cur = {}, "?", None
for r in csv.reader(txt.splitlines()):
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0].isdigit():
        cur = (fname, int(r[0]), r[1][:100])
        lines.setdefault(cur, 0.0)
        continue
    if cur and len(r) > 7 and r[0] == "" and r[2].startswith("0x"):
        try:
            lines[cur] += float(r[7])
        except ValueError:
            pass
out = [(v, f, l, src) for (f, l, src), v in lines.items()]
tot = sum(x[0] for x in out) or 1
print(f"total warp instructions {tot:.4g}")
for v, f, l, src in sorted(out, reverse=True)[:top]:
    print(f"{100 * v / tot:5.1f}% {f}:{l}  {src}")
if groups:
    acc = {}
    for v, f, l, _ in out:
        for fl, a, b, name in groups:
            if f == fl and a <= l <= b:
                acc[name] = acc.get(name, 0) + v
    for name, v in sorted(acc.items(), key=lambda x: -x[1]):
        print(f"phase {name}: {100 * v / tot:.1f}%")
