"""Probe: ECM rule quality vs m~ on the device engine (full-rule ROM as reference)."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2306_02687_b200 as F  # noqa: E402
import paper_2306_02687_b200.ecm as E  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
full = F.HyperRomModel(33, n, 0, 0)
train = np.concatenate([F.make_paths(0, 0, 24, 10), F.make_paths(1, 0, 24, 50)[:, ::5]], axis=0)
t = time.time()
X = E.force_snapshots(full, train)
Uf, S, _ = np.linalg.svd(X, full_matrices=False)
print(json.dumps({"snapshots": X.shape, "t_snap_svd": time.time() - t}), flush=True)
test = F.make_paths(0, 7, 64, 10, p0=1000)
ref_eng = F.HyperRomEngine.from_model(full)
ref_eng.alloc_points(64)
ref = [ref_eng.solve_increment(test[:, k]) for k in range(10)]
for svd_tol in (1e-4, 1e-6, 1e-8):
    k = int(np.sum(S > svd_tol * S[0]))
    for m_target in (50, 100, 200, 400):
        t = time.time()
        ids, w, res = E.ecm_select(Uf[:, :k], full.w, m_target, 1e-8)
        dt = time.time() - t
        eng = F.HyperRomEngine(full.G[ids], w, full.mat[ids], full.materials, full.volume)
        eng.alloc_points(64)
        errs = []
        for kk in range(10):
            o = eng.solve_increment(test[:, kk])
            s_ref = ref[kk]["sigma"]
            errs.append(np.linalg.norm(o["sigma"] - s_ref, axis=1).max() / np.linalg.norm(s_ref, axis=1).max())
        print(json.dumps({"svd_tol": svd_tol, "k": k, "m_target": m_target, "m": len(ids), "ecm_res": res,
                          "vol_err": abs(w.sum() - full.w.sum()), "sigma_rel_err": max(errs), "t_ecm": dt}),
              flush=True)
