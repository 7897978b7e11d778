#!/usr/bin/env python3
"""Config-1 model with each history material (J2 / power law / creep), device-resident:
python tools/mat_run.py N K P INCR PATH. Prints evals/s per material."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_02687_b200 as F  # noqa: E402

n, K, P, incr, path = (int(x) for x in sys.argv[1:6])
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(device=dev)
torch.cuda.set_stream(stream)
E = F.make_paths(path, 0, P, incr)
dE = torch.from_numpy(np.ascontiguousarray(E.transpose(1, 0, 2))).to(dev)
outs = [torch.empty(s, dtype=t, device=dev) for s, t in
        (((P, 3), torch.float64), ((P, 9), torch.float64), ((P,), torch.int32), ((P,), torch.int32),
         ((P,), torch.float64), ((P,), torch.int32))]
for name, mat in (("j2", F.J2LinearParams(1.0, 0.3, 0.01, 0.016)), ("power", F.PowerLawParams(1.0, 0.3, 0.01, 0.1)),
                  ("creep", F.CreepParams(1.0, 0.14, 0.02, 1.06, -0.56, 0.5))):
    m = F.HyperRomModel(33, n, K, 0)
    m.materials = [mat, F.ElasticParams(10.0, 0.3)]
    eng = F.HyperRomEngine.from_model(m)
    eng.set_stream(stream.cuda_stream)
    eng.alloc_points(P)
    for rep in range(2):
        eng.reset_points()
        eng.reset_stats()
        eng.set_timing(True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for k in range(incr):
            eng.solve_increment_device(dE[k].data_ptr(), *[o.data_ptr() for o in outs], stream.cuda_stream)
        e1.record(stream)
        torch.cuda.synchronize()
        st = eng.stats()
        eng.set_timing(False)
    t = e0.elapsed_time(e1) / 1e3
    print(f"{name:6s} n={n} K={K} P={P}: {P * incr / t / 1e6:.3f} M evals/s, assemblies/eval "
          f"{st['timed_assemblies'] / (P * incr):.2f}, plastic fraction "
          f"{st['timed_plastic_evals'] / max(1, st['timed_assemblies'] * m.K_j2):.2f}, failed {(outs[5].cpu().numpy() != 0).sum()}",
          flush=True)
    eng.close()
