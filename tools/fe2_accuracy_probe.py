"""FE² accuracy of the hyper-ROM against full-field HF FE² on the desk beam
(SPEC.md:507-509 method agreement; the paper's Example 1 protocol at desk
scale): HF FE² (fe2_macro_run_hf) vs hyper-ROM FE² on POD bases of growing
size from HF training trajectories (full rule, then ECM). One JSON line per case."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_02687_b200 as F  # noqa: E402
from paper_2306_02687_b200 import ecm as ECM  # noqa: E402
from paper_2306_02687_b200 import pod as P  # noqa: E402

sub = int(sys.argv[1]) if len(sys.argv) > 1 else 8
n_traj = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cfg = F.MacroConfig(u_max=0.3, n_load=10)
rve = P.HfRve(sub)
t = time.perf_counter()
hf = F.solve_program(cfg, rve)
t_hf = time.perf_counter() - t
print(json.dumps(dict(case="HF", sub=sub, steps=len(hf["U"]), macro_iters=int(hf["macro_iters"].sum()),
                      micro_iters=int(hf["micro_iters"][-1]), wall_s=t_hf, U_residual=hf["U_residual"])), flush=True)
rng = np.random.default_rng(1)
ends = rng.standard_normal((n_traj, 3))
ends *= 0.03 / np.linalg.norm(ends, axis=1, keepdims=True)
t = time.perf_counter()
X, _ = P.collect_snapshots(rve, ends, 10)
Em = rve.elastic_modes()
t_train = time.perf_counter() - t
for n in (3, 6, 12, 16, 24, 32):
    V, s, _ = P.pod_basis(X, n, Em)
    md = F.HyperRomModel(sub, K=0, basis=V)
    t = time.perf_counter()
    g = F.solve_program(cfg, F.HyperRomEngine.from_model(md))
    print(json.dumps(dict(case="hyperROM-full-rule", sub=sub, n=n, energy=P.energy_fraction(s, n - len(Em)),
                          curve_error=F.fe2.curve_error(g, hf), U_residual=g["U_residual"],
                          U_res_err=abs(g["U_residual"] - hf["U_residual"]) / cfg.u_max, wall_s=time.perf_counter() - t,
                          offline_train_s=t_train)), flush=True)
    if n in (12, 24):
        train = np.stack([P.monotonic_path(e, 10) for e in ends])  # the POD training paths
        for svd_tol in (1e-4, 1e-6):
            ids, w, res, k = ECM.build_rule(md, train, m_target=2000, tol=1e-10, svd_tol=svd_tol)
            eng = F.HyperRomEngine(md.G[ids], w, md.mat[ids], md.materials, md.volume)
            g2 = F.solve_program(cfg, eng)
            print(json.dumps(dict(case="hyperROM-ECM", sub=sub, n=n, svd_tol=svd_tol, modes=k, points=len(ids),
                                  curve_error=F.fe2.curve_error(g2, hf), curve_error_vs_rom=F.fe2.curve_error(g2, g),
                                  U_residual=g2["U_residual"])), flush=True)
