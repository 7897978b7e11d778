#!/usr/bin/env python3
"""Monolithic scheme on one device without an exchange (profiling variants):
python tools/mono_run.py N K P INCR PATH. Per increment: mono_begin, one
condensed micro iteration of every point per call (device-resident E) until
every point's relative residual is below 1e-8, mono_commit. Prints point-iterations/s."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_02687_b200 as F  # noqa: E402

n, K, P, incr, path = (int(x) for x in sys.argv[1:6])
m = F.HyperRomModel(33, n, K, 0)
eng = F.HyperRomEngine.from_model(m)
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(device=dev)  # not the legacy default stream (handle 0 = the engine's own)
torch.cuda.set_stream(stream)
eng.set_stream(stream.cuda_stream)
E = F.make_paths(path, 0, P, incr)
dE = torch.from_numpy(np.ascontiguousarray(E.transpose(1, 0, 2))).to(dev)
sig = torch.empty((P, 3), dtype=torch.float64, device=dev)
C = torch.empty((P, 9), dtype=torch.float64, device=dev)
rr = torch.empty(P, dtype=torch.float64, device=dev)
pc = torch.empty(P, dtype=torch.int32, device=dev)
st = torch.empty(P, dtype=torch.int32, device=dev)
eng.alloc_points(P)
for rep in range(2):
    eng.reset_points()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    its = 0
    for k in range(incr):
        eng.mono_begin()
        for it in range(30):
            eng.mono_iterate_device(dE[k].data_ptr(), sig.data_ptr(), C.data_ptr(), rr.data_ptr(), pc.data_ptr(),
                                    st.data_ptr(), stream.cuda_stream)
            its += 1
            if float(rr.max()) <= 1e-8 and int(st.abs().max()) == 0:
                break
        eng.mono_commit()
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    print(f"mono n={n} K={K} P={P}: {P * its / t / 1e6:.3f} M point-iterations/s, {its} iterations, "
          f"{P * incr / t / 1e6:.3f} M evals/s", flush=True)
