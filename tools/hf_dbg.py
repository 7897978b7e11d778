import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_02687_b200 as F
from paper_2306_02687_b200 import pod as P
rve = P.HfRve(int(sys.argv[1]) if len(sys.argv) > 1 else 8)
rng = np.random.default_rng(0)
ends = rng.standard_normal((6, 3)); ends *= 0.02 / np.linalg.norm(ends, axis=1, keepdims=True)
paths = np.stack([P.monotonic_path(e, 8) for e in ends])
for rep in range(3):
    r = rve.trajectories(paths)
    print(rep, r["status"], F.hrom.lib.fe2_last_error().decode(), flush=True)
