"""Desk-beam FE² run, nested vs monolithic scheme, on the device engine:
steps, macro iterations, micro iterations, wall time, U_res. One JSON line
per scheme."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_02687_b200 as F  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
m = F.HyperRomModel(33, n, 200, 0)
for scheme in ("nested", "monolithic"):
    F.solve_program(F.MacroConfig(u_max=0.02, n_load=2, scheme=scheme), F.HyperRomEngine.from_model(m))  # warm-up
    g = F.solve_program(F.MacroConfig(u_max=0.3, n_load=10, scheme=scheme), F.HyperRomEngine.from_model(m))
    print(json.dumps(dict(scheme=scheme, n=n, steps=len(g["U"]), macro_iters=int(g["macro_iters"].sum()),
                          micro_iters=int(g["micro_iters"][-1]), wall_ms=float(g["wall_ms"][-1]),
                          U_residual=g["U_residual"], R_peak=float(g["R"].max()))))
