#!/usr/bin/env python3
"""Throughput / roofline sweep over BASELINE.json configs on one B200.

config 4: n in {8,16,32,64,128} x K in {100,400,1000,4000}, config-0 path
generator, 5 increments; config 0 (1,024 points, 20 increments); config 3 at
a reduced point count (n = 64, K = 2,000, 20 increments). Points per cell are
scaled so each timed trajectory takes about `--seconds` (P <= the config's P).
Prints one JSON object per cell (evals/s, assemblies per eval, plastic
fraction, algorithmic TFLOP/s vs the measured DMMA peak, history GB/s).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2306_02687_b200 as F  # noqa: E402

DMMA_PEAK = json.load(open(os.path.join(ROOT, "profiles", "r01_fp64_peak.json")))["dmma_tflops_w16"]
try:
    HBM = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:
    HBM = 6650.0


def run_cell(name, n, K, P_max, incr, path, seconds, seed=0, points=0):
    import torch

    fs = path == 2  # finite strain (config 2)
    nc, nt = (4, 16) if fs else (3, 9)
    m = F.HyperRomModel(33, n, K, seed)
    eng = F.HyperRomEngine.from_model(m, finite_strain=fs)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(device=dev)  # not the legacy default stream (handle 0 = the engine's own)
    torch.cuda.set_stream(stream)
    eng.set_stream(stream.cuda_stream)

    def trajectory(P):
        E = F.make_paths(path, seed, P, incr)
        dE = torch.from_numpy(np.ascontiguousarray(E.transpose(1, 0, 2))).to(dev)
        outs = [torch.empty(s, dtype=t, device=dev) for s, t in
                (((P, nc), torch.float64), ((P, nt), torch.float64), ((P,), torch.int32), ((P,), torch.int32),
                 ((P,), torch.float64), ((P,), torch.int32))]
        eng.alloc_points(P)
        eng.reset_stats()
        eng.set_timing(True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for k in range(incr):
            eng.solve_increment_device(dE[k].data_ptr(), outs[0].data_ptr(), outs[1].data_ptr(), outs[2].data_ptr(),
                                       outs[3].data_ptr(), outs[4].data_ptr(), outs[5].data_ptr(), stream.cuda_stream)
        e1.record(stream)
        torch.cuda.synchronize()
        eng.set_timing(False)
        st = outs[5].cpu().numpy()
        return e0.elapsed_time(e1) / 1e3, eng.stats(), int((st != 0).sum()), outs[2].cpu().numpy()

    P = min(P_max, 1024)
    trajectory(P)  # warm-up (module load, first launch)
    t, _, _, _ = trajectory(P)
    P = int(min(P_max, max(256, P * seconds / max(t, 1e-3)))) if not points else points
    t, s, failed, iters_sum = trajectory(P)
    K_j2 = m.K_j2
    evals = P * incr
    # SURVEY §8(d) flops: small strain 3 n (n+9) per CONTRACTED cubature point (the plastic
    # J2 points; the elastic block is precomputed), finite strain 8 n (n+5) per cubature point
    kms = s["kernel_ms"]
    if fs:
        flops = s["timed_assemblies"] * 8.0 * K * n * (n + 5)
        equiv = flops
    else:
        flops = s["timed_plastic_evals"] * 3.0 * n * (n + 9)
        equiv = s["timed_assemblies"] * 3.0 * K_j2 * n * (n + 9)  # as if every J2 point were contracted
    # DRAM history stream: one committed read + one candidate write (40 B each) per J2 point
    # per launch (double-buffered history; L2 hits excluded)
    hbm_bytes = s["timed_launches"] * P * K_j2 * 80.0
    return {
        "cell": name, "n": n, "K": K, "K_j2": K_j2, "points": P, "increments": incr, "failed": failed,
        "evals_per_s": evals / t, "ms": t * 1e3,
        "assemblies_per_eval": s["timed_assemblies"] / evals,
        "plastic_fraction": s["timed_plastic_evals"] / max(1, s["timed_assemblies"] * K_j2),
        "newton_iters_last_incr": float(np.mean(iters_sum)),
        "contracted_tflops": flops / (kms / 1e3) / 1e12,
        "frac_of_dmma_peak": flops / (kms / 1e3) / 1e12 / DMMA_PEAK,
        "algorithmic_equiv_frac": equiv / (kms / 1e3) / 1e12 / DMMA_PEAK,
        "history_gbs": hbm_bytes / (kms / 1e3) / 1e9, "frac_of_hbm": hbm_bytes / (kms / 1e3) / 1e9 / HBM,
        "kernel_share": kms / (t * 1e3),
        "kernel_evals_per_s": evals / (kms / 1e3),
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=2.0)
    ap.add_argument("--which", default="0,3,4")
    ap.add_argument("--only", default="", help="comma-separated substrings of cell names to run")
    ap.add_argument("--points", type=int, default=0, help="fixed point count per cell (0 = scale to --seconds)")
    ap.add_argument("--full", action="store_true", help="every cell at its BASELINE point count (config 4: 131,072)")
    args = ap.parse_args()
    which = set(args.which.split(","))
    cells = []
    if "0" in which:
        cells.append(("config0", 12, 200, 1024, 20, 0))
    if "2" in which:
        cells.append(("config2", 32, 600, 262144, 30, 2))
    if "3" in which:
        cells.append(("config3_subset", 64, 2000, 1048576, 20, 0))
    if "4" in which:
        for n in (8, 16, 32, 64, 128):
            for K in (100, 400, 1000, 4000):
                cells.append((f"config4_n{n}_K{K}", n, K, 131072, 5, 0))
    if args.only:
        keys = args.only.split(",")
        cells = [c for c in cells if any(k in c[0] for k in keys)]
    for c in cells:
        t0 = time.time()
        r = run_cell(*c, seconds=args.seconds, points=c[3] if args.full else args.points)
        r["wall_s"] = time.time() - t0
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
