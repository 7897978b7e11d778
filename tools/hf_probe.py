"""Timing probe of the offline HF + POD stage on the device (SURVEY §8(f)
rank 2): one 20-step HF trajectory on default_cell(sub), the elastic modes,
and the POD of n_traj trajectories' snapshots. Prints one JSON line."""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_02687_b200 import pod as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sub", type=int, default=33)
ap.add_argument("--n-traj", type=int, default=4)
ap.add_argument("--n-steps", type=int, default=20)
ap.add_argument("--modes", type=int, default=12)
a = ap.parse_args()

t0 = time.perf_counter()
rve = P.HfRve(a.sub)
t1 = time.perf_counter()
rng = np.random.default_rng(0)
ends = rng.standard_normal((a.n_traj, 3))
ends *= 0.02 / np.linalg.norm(ends, axis=1, keepdims=True)
cols, iters, per = [], 0, []
for e in ends:
    s = time.perf_counter()
    r = rve.trajectory(P.monotonic_path(e, a.n_steps))
    per.append(time.perf_counter() - s)
    cols.append(r["snapshots"])
    iters += int(r["iterations"].sum())
t2 = time.perf_counter()
Em = rve.elastic_modes()
t3 = time.perf_counter()
X = np.concatenate(cols)
V, sv, mx = P.pod_basis(X, a.modes, Em)
t4 = time.perf_counter()
P.pod_basis(X, a.modes, Em)
t5 = time.perf_counter()
print(json.dumps(dict(sub=a.sub, n_dofs=rve.n_dofs, n_free=rve.n_free, n_ips=rve.n_ips, create_s=t1 - t0,
                      trajectories=a.n_traj, steps=a.n_steps, newton_iters=iters, traj_s=per,
                      s_per_newton_iter=(t2 - t1) / max(iters, 1), elastic_modes_s=t3 - t2, pod_s=t4 - t3, pod_again_s=t5 - t4,
                      snapshots=X.shape, energy_at_modes=P.energy_fraction(sv, a.modes - len(Em)), max_modes=mx)))
