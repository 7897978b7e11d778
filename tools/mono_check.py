#!/usr/bin/env python3
"""Determinism / cross-variant check of the monolithic iteration at scale:
runs INCR increments x ITERS fixed iterations and saves (sigma, C, rel_res)
of every iteration to OUT.npz."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_02687_b200 as F  # noqa: E402

n, K, P, incr, path, iters = (int(x) for x in sys.argv[1:7])
out = sys.argv[7]
m = F.HyperRomModel(33, n, K, 0)
eng = F.HyperRomEngine.from_model(m)
E = F.make_paths(path, 0, P, incr)
eng.alloc_points(P)
rec = []
for k in range(incr):
    eng.mono_begin()
    for it in range(iters):
        o = eng.mono_iterate(np.ascontiguousarray(E[:, k]))
        rec.append(np.concatenate([o["sigma"], o["C"].reshape(P, 9), o["rel_res"][:, None],
                                   o["status"][:, None].astype(float)], 1))
    eng.mono_commit()
np.savez(out, r=np.stack(rec))
print("saved", out, flush=True)
