#!/usr/bin/env python3
"""Run one BASELINE config (or an (n, K) cell) device-resident for profiling:
python tools/cfg_run.py N K P INCR PATH [REPEAT]. Prints evals/s per repeat
(CUDA events on the engine's stream). FE2_LIB selects a tuning-variant library
(e.g. -DFE2_INC_PROF / -DFE2_BIG_PROF builds print their phase timelines)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_02687_b200 as F  # noqa: E402

n, K, P, incr, path = (int(x) for x in sys.argv[1:6])
rep = int(sys.argv[6]) if len(sys.argv) > 6 else 1
m = F.HyperRomModel(33, n, K, 0)
fs = path == 2  # finite-strain Biot variant (config 2): H (4) in, P (4) and A (16) out
eng = F.HyperRomEngine.from_model(m, finite_strain=fs)
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(device=dev)  # not the legacy default stream (handle 0 = the engine's own)
torch.cuda.set_stream(stream)
eng.set_stream(stream.cuda_stream)
E = F.make_paths(path, 0, P, incr)
dE = torch.from_numpy(np.ascontiguousarray(E.transpose(1, 0, 2))).to(dev)
outs = [torch.empty(s, dtype=t, device=dev) for s, t in
        (((P, 4 if fs else 3), torch.float64), ((P, 16 if fs else 9), torch.float64), ((P,), torch.int32), ((P,), torch.int32),
         ((P,), torch.float64), ((P,), torch.int32))]
eng.alloc_points(P)
for r in range(rep):
    eng.reset_points()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for k in range(incr):
        eng.solve_increment_device(dE[k].data_ptr(), *[o.data_ptr() for o in outs], stream.cuda_stream)
    e1.record(stream)
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3
    st = outs[5].cpu().numpy()
    print(f"n={n} K={K} P={P} incr={incr}: {P * incr / t / 1e6:.3f} M evals/s ({t * 1e3:.1f} ms), failed {(st != 0).sum()}",
          flush=True)
