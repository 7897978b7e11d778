"""ROM -> HF convergence probe: POD bases of growing size from HF training
trajectories, hyper-ROM (full rule) vs HF on unseen paths. One JSON line per case."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_02687_b200 as F  # noqa: E402
from paper_2306_02687_b200 import pod as P  # noqa: E402

sub = int(sys.argv[1]) if len(sys.argv) > 1 else 12
rve = P.HfRve(sub)
Em = rve.elastic_modes()
tests = [np.array([0.012, -0.006, 0.010]), np.array([0.02, 0.0, 0.0]), np.array([-0.01, 0.015, -0.005])]
hf = [rve.trajectory(np.stack([t * k / 10 for k in range(1, 11)]), snapshots=False)["sigma"] for t in tests]
for n_traj in (10, 30):
    rng = np.random.default_rng(1)
    ends = rng.standard_normal((n_traj, 3))
    ends *= 0.025 / np.linalg.norm(ends, axis=1, keepdims=True)
    X, _ = P.collect_snapshots(rve, ends, 10)
    for n in (3, 6, 8, 12, 16, 24, 32):
        V, s, _ = P.pod_basis(X, n, Em)
        md = F.HyperRomModel(sub, K=0, basis=V)
        errs = []
        for t, h in zip(tests, hf):
            eng = F.HyperRomEngine.from_model(md)
            eng.alloc_points(1)
            sig = np.stack([eng.solve_increment((t * k / 10)[None])["sigma"][0] for k in range(1, 11)])
            errs.append(float(np.linalg.norm(sig - h) / np.linalg.norm(h)))
        print(json.dumps(dict(sub=sub, n_traj=n_traj, n=n, energy=P.energy_fraction(s, n - len(Em)), errs=errs)),
              flush=True)
