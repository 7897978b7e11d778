"""Run one (n, K) model for a few increments (watchdog on) — debugging aid."""
import sys
import time

import numpy as np

import paper_2306_02687_b200 as F

n, K, P, incr = (int(x) for x in sys.argv[1:5])
m = F.HyperRomModel(33, n, K, 0)
E = F.make_paths(0, 0, P, incr)
eng = F.HyperRomEngine.from_model(m)
eng.alloc_points(P)
for k in range(incr):
    t = time.time()
    o = eng.solve_increment(E[:, k])
    print(k, "%.3f s" % (time.time() - t), int(o["iters"].sum()), int((o["status"] != 0).sum()), flush=True)
