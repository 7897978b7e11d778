"""Timing probe of the offline HF + POD stage on the device (SURVEY §8(f)
rank 2): n_traj 20-step HF training trajectories on default_cell(sub), one
after another (fe2_hf_trajectory) and as one concurrent batch
(fe2_hf_trajectories), the elastic modes and the POD. Prints one JSON line."""
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
ap.add_argument("--n-traj", type=int, default=40)
ap.add_argument("--n-steps", type=int, default=20)
ap.add_argument("--modes", type=int, default=12)
ap.add_argument("--serial", type=int, default=2, help="trajectories timed one after another")
a = ap.parse_args()

t0 = time.perf_counter()
rve = P.HfRve(a.sub)
t1 = time.perf_counter()
rng = np.random.default_rng(0)
ends = rng.standard_normal((a.n_traj, 3))
ends *= 0.02 / np.linalg.norm(ends, axis=1, keepdims=True)
paths = np.stack([P.monotonic_path(e, a.n_steps) for e in ends])
per, iters_serial = [], 0
for e in paths[:a.serial]:
    s = time.perf_counter()
    r = rve.trajectory(e)
    per.append(time.perf_counter() - s)
    iters_serial += int(r["iterations"].sum())
t2 = time.perf_counter()
rb = rve.trajectories(paths)
t3 = time.perf_counter()
Em = rve.elastic_modes()
t4 = time.perf_counter()
X = rb["snapshots"].reshape(-1, rve.n_dofs)
V, sv, mx = P.pod_basis(X, a.modes, Em)
t5 = time.perf_counter()
iters = int(rb["iterations"].sum())
print(json.dumps(dict(sub=a.sub, n_dofs=rve.n_dofs, n_free=rve.n_free, n_ips=rve.n_ips,
                      half_bandwidth=rve.half_bandwidth, create_s=t1 - t0, trajectories=a.n_traj, steps=a.n_steps,
                      serial_traj_s=per, serial_s_per_newton_iter=(t2 - t1) / max(iters_serial, 1),
                      batch_s=t3 - t2, batch_newton_iters=iters, batch_status_failed=int((rb["status"] != 0).sum()),
                      batch_traj_per_s=a.n_traj / (t3 - t2), elastic_modes_s=t4 - t3, pod_s=t5 - t4,
                      training_total_s=t5 - t2, snapshots=X.shape,
                      energy_at_modes=P.energy_fraction(sv, a.modes - len(Em)), max_modes=mx)))
