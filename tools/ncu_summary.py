#!/usr/bin/env python3
"""Summarise ncu captures into the JSON kept under profiles/.

  ncu_summary.py full  REPORT.ncu-rep  OUT.json [--label L]   (one --set full capture)
  ncu_summary.py launches LAUNCHES.csv OUT.json                (--metrics gpu__time_duration.sum list)
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = {
    "duration_ns": "gpu__time_duration.sum",
    "dram_bytes_read": "dram__bytes_read.sum",
    "dram_bytes_write": "dram__bytes_write.sum",
    "sm_cycles_active": "sm__cycles_active.avg",
    "dmma_pipe_pct_active": "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "fp64_pipe_pct_active": "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "lsu_pipe_pct_active": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "registers_per_thread": "launch__registers_per_thread",
    "grid_size": "launch__grid_size",
    "block_size": "launch__block_size",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smem_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "local_spill_bytes": "l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum",
}


def _num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return x


def full(report, out, label):
    raw = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u, v = rows[0], rows[1], rows[2]
    d = dict(zip(h, v))
    res = {"label": label, "report": report, "kernel": d.get("Kernel Name")}
    for k, m in KEYS.items():
        if m in d:
            res[k] = _num(d[m])
    if "dram_bytes_read" in res and "dram_bytes_write" in res:
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        ur = u[h.index(KEYS["dram_bytes_read"])]
        uw = u[h.index(KEYS["dram_bytes_write"])]
        res["dram_bytes_per_launch"] = res["dram_bytes_read"] * scale.get(ur, 1) + res["dram_bytes_write"] * scale.get(uw, 1)
        res["dram_units"] = [ur, uw]
    stalls = {}
    for name, val in zip(h, v):
        if "pcsamp_warps_issue_stalled" in name and not name.endswith("not_issued"):
            x = _num(val)
            if isinstance(x, float):
                stalls[name.replace("smsp__pcsamp_warps_issue_stalled_", "")] = x
    tot = sum(stalls.values()) or 1.0
    res["stall_share"] = {k: round(x / tot, 4) for k, x in sorted(stalls.items(), key=lambda t: -t[1])[:8]}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


def _short_name(full):
    """'void ns::<unnamed>::k_increment<3, 8, 1, 0>(ns::IncArgs)' -> 'k_increment'."""
    s = full.strip()
    if s.endswith(")"):  # drop the (balanced) argument list
        depth = 0
        for i in range(len(s) - 1, -1, -1):
            depth += {")": 1, "(": -1}.get(s[i], 0)
            if depth == 0:
                s = s[:i]
                break
    if s.endswith(">"):  # drop the (balanced) template arguments
        depth = 0
        for i in range(len(s) - 1, -1, -1):
            depth += {">": 1, "<": -1}.get(s[i], 0)
            if depth == 0:
                s = s[:i]
                break
    return s.replace("::", " ").split()[-1] if s.strip() else full


def launches(path, out):
    text = open(path).read()
    lines = [ln for ln in text.splitlines() if ln.startswith('"')]
    rows = list(csv.reader(lines))
    h = rows[0]
    ik, im, iv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if r[im] != "gpu__time_duration.sum":
            continue
        name = _short_name(r[ik])
        agg[name][0] += 1
        agg[name][1] += _num(r[iv])
    tot = sum(t for _, t in agg.values()) or 1.0
    res = {"source": path, "note": "cold-cache, serialised ncu launch list: use shares, not absolute times",
           "kernels": {k: {"launches": c, "total": t, "share": t / tot} for k, (c, t) in
                       sorted(agg.items(), key=lambda kv: -kv[1][1])}}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    mode, src, dst = sys.argv[1:4]
    lab = sys.argv[sys.argv.index("--label") + 1] if "--label" in sys.argv else ""
    full(src, dst, lab) if mode == "full" else launches(src, dst)
