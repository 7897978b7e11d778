import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_02687_b200 as F
from paper_2306_02687_b200 import pod as P
for umax, nl in ((0.2, 4), (0.2, 8)):
    cfg = F.MacroConfig(u_max=umax, n_load=nl, max_unload=2 * nl)
    a = F.solve_program(cfg, P.HfRve(8))
    cfg_m = F.MacroConfig(u_max=umax, n_load=nl, max_unload=2 * nl, scheme="monolithic")
    b = F.solve_program(cfg_m, P.HfRve(8))
    print(umax, nl, "nested iters", a["macro_iters"], "micro", a["micro_iters"][-1], "R", a["R"])
    print(umax, nl, "mono   iters", b["macro_iters"], "micro", b["micro_iters"][-1], "R", b["R"])
    print("  max rel R diff", np.abs(a["R"] - b["R"]).max() / np.abs(a["R"]).max(), "Ures", a["U_residual"], b["U_residual"])
