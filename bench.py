#!/usr/bin/env python3
"""Benchmark: macro Gauss-point hyper-ROM evaluations/sec (fp64) on B200.

One evaluation = one macro Gauss point advanced by one load increment to
reduced-Newton convergence, returning Σ and the condensed C_macro
(BASELINE.md). A bench "step" is one full BASELINE config-1 trajectory of the
per-rank batch: P = 65,536 points x 50 increments (n = 24 modes, K = 400
cubature points, seeded reversal paths), from the virgin state. Weak scaling
over ranks: every rank owns P points (global ids rank*P..), and after every
increment the macro stress, condensed tangent, residual norms and status are
all-gathered over NCCL (the monolithic scheme's exchange).

  monolithic : the paper's scheme on the same workload — one condensed reduced
           Newton iteration of every point per macro iteration, the NCCL
           exchange after EVERY iteration, lockstep termination (also at N = 1,
           one-rank communicator).
  extra_configs : config 2 (finite strain), config 4's full-size roofline sweep
           (20 cells of 131,072 points, one GPU) and config 3 (1,048,576 points,
           n = 64, K = 2,000, split over the ranks: strong scaling) with their
           own rooflines; config 3 also runs the monolithic scheme with the
           per-iteration exchange (the north_star scaling run).

  value  : device-resident inputs (all increments' E already in HBM),
           CUDA events on the engine's stream, max over ranks.
  e2e    : the host-buffer C-ABI call fe2_hrom_solve_increment per increment
           (pinned E H2D + outputs D2H inside the timed region).
  --impl reference : the reference CPU algorithm (the C++ oracle restatement,
           oracle/) on all host cores, bounded sample of the same workload.
"""
import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # BASELINE.json configs[1]: the metric's quoted workload (fits one GPU)
    1: dict(name="config1_beam_small_strain_j2", P=65536, n=24, K=400, incr=50, path=1, subdivisions=33),
    # configs[0]: the reference's CPU-runnable case (parity config)
    0: dict(name="config0_small_strain_j2", P=1024, n=12, K=200, incr=20, path=0, subdivisions=33),
    # configs[2]: finite-strain Biot J2 (parity unpinned: no reference code)
    2: dict(name="config2_finite_strain_biot_j2", P=262144, n=32, K=600, incr=30, path=2, subdivisions=33),
    # configs[3]: the multi-GPU case — P is the TOTAL point count, split over the ranks
    # (strong scaling); n = 64 runs the CTA-per-point kernel. ~2 min per step on one GPU.
    3: dict(name="config3_multi_gpu", P=1048576, n=64, K=2000, incr=20, path=0, subdivisions=33, strong=True),
}
METRIC = "macro Gauss-point hyper-ROM evaluations/sec (fp64)"
UNIT = "evals/s"
DMMA_PEAK_FILE = os.path.join(ROOT, "profiles", "r01_fp64_peak.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-mono", dest="mono", action="store_false",
                    help="skip the monolithic-scheme runs (per-iteration exchange, lockstep termination)")
    ap.add_argument("--config", type=int, default=1, choices=sorted(CONFIGS))
    ap.add_argument("--points", type=int, default=0, help="override points per rank (debug)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-points", type=int, default=0)
    ap.add_argument("--constitutive-points", type=int, default=1 << 25,
                    help="material points of the SoA constitutive-update roofline run (0 = skip)")
    ap.add_argument("--extra-configs", default="2,3,4",
                    help="comma-separated configs also timed device-resident (2-increment warm-up + 1 step) "
                         "into extra_configs of the line; config 3 adds its monolithic run; '' to skip")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def flops_per_assembly(n, K_j2, K=0, finite=False):
    if finite:
        # F_asm = 8 K n (n + 5) — every cubature point,
        # the full non-symmetric K_aa, K_aF (n x 4) and r
        return 8.0 * K * n * (n + 5)
    # F_asm = 3 K n (n + 9) (upper-triangle K_aa + K_aE + r),
    # K = the J2 cubature points actually contracted (elastic block precomputed)
    return 3.0 * K_j2 * n * (n + 9)


class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.p is not None:
            self.p.terminate()
            try:
                out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.p.kill()
                out, _ = self.p.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def wrap_dev(ptr, shape, typestr, dev):
    """torch view of a device buffer owned by the native engine."""
    import torch

    class _Buf:
        __cuda_array_interface__ = {"shape": shape, "typestr": typestr, "data": (ptr, False), "version": 3,
                                    "strides": None, "stream": None}

    return torch.as_tensor(_Buf(), device=dev)


def cpu_reference_run(cfg, n_points, threads, seed=0):
    """The reference CPU algorithm (oracle restatement) on a sample of the
    workload: the first n_points points, all increments. Returns evals/s."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as O
    m = O.Model(cfg["subdivisions"], cfg["n"], cfg["K"], seed)
    mats = [("j2", 1.0, 0.3, 0.01, 0.016), ("elastic", 10.0, 0.3)]
    if cfg["path"] == 2:
        E = O.paths_fs(seed, n_points, cfg["incr"])
        G4 = O.model_g4(cfg["subdivisions"], cfg["n"], cfg["K"], seed)
        h = O.HromFs(G4, m.w, m.mat, mats, m.volume)
    else:
        E = O.paths(cfg["path"], seed, n_points, cfg["incr"])
        h = O.Hrom(m.G, m.w, m.mat, mats, m.volume)
    t0 = time.perf_counter()
    r = h.run(E, threads=threads)
    dt = time.perf_counter() - t0
    assert (r["status"] == 0).all()
    return n_points * cfg["incr"] / dt, dt


def calibrate_cpu_points(cfg, threads, seconds):
    """Sample size (points, all increments) giving about `seconds` of CPU work."""
    n0 = max(2 * threads, 16)
    v0, _ = cpu_reference_run(cfg, n0, threads)
    return int(max(n0, min(1 << 16, v0 * seconds / cfg["incr"])))


def run_reference(args, cfg):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    n_pts = args.cpu_sample_points or calibrate_cpu_points(cfg, threads, seconds=8.0)
    for _ in range(args.warmup):
        cpu_reference_run(cfg, max(threads, 16), threads)
    vals, times = [], []
    for _ in range(args.steps):
        v, dt = cpu_reference_run(cfg, n_pts, threads)
        vals.append(v)
        times.append(dt)
    value = float(np.mean(vals))
    sample = f"first {n_pts} points x {cfg['incr']} increments of {cfg['name']} per step"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(times)),
        "higher_is_better": True, "scaling": "strong" if cfg.get("strong") else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["name"], "points": n_pts, "modes": cfg["n"], "cubature": cfg["K"],
                   "increments": cfg["incr"]},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config4_sweep():
    """BASELINE configs[4]: n in {8,16,32,64,128} x K in {100,400,1000,4000}, 131,072 points
    x 5 increments each at full size (tools/sweep.py run_cell: one untimed P = 1,024
    trajectory, then the timed one; CUDA events on the engine's stream). Per cell:
    evals/s, the fraction of the DMMA peak on the contracted (plastic) points, the
    DRAM history rate against HBM — the crossover the config asks for."""
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import sweep
    cells = {}
    for n in (8, 16, 32, 64, 128):
        for K in (100, 400, 1000, 4000):
            r = sweep.run_cell(f"n{n}_K{K}", n, K, 131072, 5, 0, seconds=1.0, points=131072)
            if r["failed"]:
                raise SystemExit(f"bench: config 4 cell n={n} K={K}: {r['failed']} points failed")
            cells[f"n{n}_K{K}"] = {k: r[k] for k in ("evals_per_s", "ms", "assemblies_per_eval", "plastic_fraction",
                                                     "frac_of_dmma_peak", "algorithmic_equiv_frac", "frac_of_hbm",
                                                     "history_gbs")}
    return {"workload": "config4: 131,072 points x 5 increments per cell, config-0 path generator",
            "unit": UNIT, "cells": cells}


def rank_points(cfg, ws, rank):
    """(points on this rank, first global point id): weak scaling gives every rank
    cfg["P"] points; a strong-scaling config splits cfg["P"] in contiguous blocks."""
    if cfg.get("strong"):
        per = (cfg["P"] + ws - 1) // ws
        lo = min(cfg["P"], rank * per)
        return min(per, cfg["P"] - lo), lo
    return cfg["P"], rank * cfg["P"]


COMM = [None]  # this rank's NCCL communicator (fe2_nccl_comm_init), N > 1


class DeviceRun:
    """One config on this rank: model, engine, device-resident path and outputs."""

    def __init__(self, F, torch, cfg, rank, local, dev, stream, ws=1):
        self.cfg, self.dev, self.stream, self.torch = cfg, dev, stream, torch
        self.finite = cfg["path"] == 2
        self.nc, self.nt = (4, 16) if self.finite else (3, 9)
        P, p0 = rank_points(cfg, ws, rank)
        incr = cfg["incr"]
        self.P = P
        self.model = F.HyperRomModel(cfg["subdivisions"], cfg["n"], cfg["K"], seed=0)
        E_host = F.make_paths(cfg["path"], 0, P, incr, p0=p0)  # (P, incr, nc), global-id streams
        self.E_inc = np.ascontiguousarray(E_host.transpose(1, 0, 2))  # (incr, P, nc)
        self.eng = F.HyperRomEngine.from_model(self.model, device=local, finite_strain=self.finite)
        self.eng.alloc_points(P)
        self.eng.set_stream(stream.cuda_stream)
        f64, i32 = torch.float64, torch.int32
        self.dE = torch.from_numpy(self.E_inc).to(dev)
        self.d_sig = torch.empty((P, self.nc), dtype=f64, device=dev)
        self.d_C = torch.empty((P, self.nt), dtype=f64, device=dev)
        self.d_res = torch.empty(P, dtype=f64, device=dev)
        self.d_it = torch.empty(P, dtype=i32, device=dev)
        self.d_pc = torch.empty(P, dtype=i32, device=dev)
        self.d_st = torch.empty(P, dtype=i32, device=dev)
        self.width = self.nc + self.nt + 2
        self.steps_timed = 1
        self.pack = torch.empty((P, self.width), dtype=f64, device=dev)
        self.gathered = None

    def gather(self, dist, ws, sig, C, res, st):
        """The monolithic scheme's exchange: all-gather (Σ | P, C | A, residual
        norm, status) of every point over NCCL through the engine's C ABI
        (fe2_hrom_gather: device-side packing into this rank's block,
        in-place ncclAllGather, max all-reduce of the failure flag)."""
        if ws == 1:
            return
        self.ensure_gather_buffer()
        self.any_failed = self.eng.gather(COMM[0], self.gathered.data_ptr(), sig.data_ptr(), C.data_ptr(),
                                          res.data_ptr(), st.data_ptr())

    def ensure_gather_buffer(self):
        """[world][P_max][width] device buffer of the exchange (fe2_hrom_gather_layout:
        ranks may hold different point counts; their blocks are padded to P_max)."""
        if self.gathered is None:
            p_max, self.counts = self.eng.gather_layout(COMM[0])
            self.gathered = self.torch.empty((COMM[0].nranks, p_max, self.width), dtype=self.pack.dtype,
                                             device=self.dev)

    def mono_step(self, tol=1e-8, max_iter=30):
        """The monolithic scheme with the exchange after EVERY Newton iteration (SURVEY
        §8(e), BASELINE config 3): per load increment, fe2_hrom_mono_begin, then
        fe2_hrom_mono_iterate_device (one condensed reduced-Newton iteration of every point,
        device-resident E) followed by fe2_hrom_gather of {Σ, C_macro, ‖r‖, status} of all
        points over NCCL with the max all-reduce of "some point failed" / "some point above
        tol" — lockstep termination when no point on any rank is above tol — then
        fe2_hrom_mono_commit. Returns the number of iterations of each increment."""
        self.eng.reset_points()
        self.ensure_gather_buffer()
        its = []
        for k in range(self.cfg["incr"]):
            self.eng.mono_begin()
            for it in range(1, max_iter + 1):
                self.eng.mono_iterate_device(self.dE[k].data_ptr(), self.d_sig.data_ptr(), self.d_C.data_ptr(),
                                             self.d_res.data_ptr(), self.d_pc.data_ptr(), self.d_st.data_ptr(),
                                             self.stream.cuda_stream)
                failed, above = self.eng.gather(COMM[0], self.gathered.data_ptr(), self.d_sig.data_ptr(),
                                                self.d_C.data_ptr(), self.d_res.data_ptr(), self.d_st.data_ptr(),
                                                res_tol=tol, flags=True)
                if failed:
                    raise SystemExit(f"bench: monolithic iteration failed ({self.cfg['name']}, increment {k})")
                if not above:
                    break
            else:
                raise SystemExit(f"bench: monolithic iteration not converged in {max_iter} ({self.cfg['name']})")
            its.append(it)
            self.eng.mono_commit()
        return its

    def device_step(self, dist, ws, n_incr=None):
        self.eng.reset_points()
        for k in range(self.cfg["incr"] if n_incr is None else n_incr):
            self.eng.solve_increment_device(self.dE[k].data_ptr(), self.d_sig.data_ptr(), self.d_C.data_ptr(),
                                            self.d_it.data_ptr(), self.d_pc.data_ptr(), self.d_res.data_ptr(),
                                            self.d_st.data_ptr(), self.stream.cuda_stream)
            self.gather(dist, ws, self.d_sig, self.d_C, self.d_res, self.d_st)

    def check_converged(self):
        st = self.d_st.cpu().numpy()
        if (st != 0).any():
            raise SystemExit(f"bench: {int((st != 0).sum())} points of {self.cfg['name']} failed to converge")

    def roofline(self, stats, ms, peak, peak_src):
        """F_asm = 3 K n (n+9) per point-assembly with K = the cubature points
        the kernel actually contracts. The increment kernels contract only the plastic J2
        points (elastic-predictor split), so `achieved` counts
        timed_plastic_evals x 3 n (n+9); the count as if every J2 point were contracted is
        kept under `algorithmic_equiv` (not a roofline claim). Config 2 contracts every
        cubature point: 8 K n (n+5)."""
        cfg, model = self.cfg, self.model
        n, K_j2 = cfg["n"], model.K_j2
        kms = stats["kernel_ms"]
        nt = (n + 7) // 8
        equiv = None
        if self.finite:  # every cubature point: NT^2 + NT DMMA.8x8x4 (512 flop) per point-assembly
            F_asm = flops_per_assembly(n, K_j2, cfg["K"], True)
            flops = stats["timed_assemblies"] * F_asm
            executed = stats["timed_assemblies"] * cfg["K"] * (nt * nt + nt) * 512
            kernel = "k_increment_fs (persistent: Biot update + DMMA k-step per cubature point + warp LU/Newton/condensation + commit)"
            definition = "SURVEY §8(d) config 2: F_asm = 8 K n (n+5) per point-assembly (all cubature points contracted)"
        else:  # every plastic point = 3 k-entries = 0.75 k-steps of NT(NT+1)/2 DMMA.8x8x4
            flops = stats["timed_plastic_evals"] * 3.0 * n * (n + 9)
            executed = stats["timed_plastic_evals"] * 0.75 * (nt * (nt + 1) // 2) * 512
            kernel = ("k_increment (persistent: DMMA hyper-assembly + warp Cholesky/Newton/condensation + commit)"
                      if n <= 32 else
                      "k_increment_big (persistent, CTA per point: staged-B DMMA hyper-assembly + CTA Cholesky/"
                      "Newton/condensation)")
            definition = ("SURVEY §8(d) F_asm = 3 K n (n+9) per point-assembly, K = the plastic J2 points the "
                          "kernel contracts (elastic points enter through the precomputed elastic block)")
            F_asm = 3.0 * K_j2 * n * (n + 9)
            if kms:
                eq = stats["timed_assemblies"] * F_asm / (kms / 1e3) / 1e12
                equiv = {"achieved": eq, "frac": eq / peak, "flops_per_point_assembly": F_asm,
                         "note": "3 K_J2 n (n+9): as if every J2 point were contracted; the elastic-predictor "
                                 "split does that work once per model, so this is throughput-equivalent only"}
        achieved = flops / (kms / 1e3) / 1e12 if kms else None
        launches_t = max(1, stats["timed_launches"])
        return {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": (achieved / peak) if achieved else None, "kernel": kernel, "peak_source": peak_src,
                "flops_definition": definition, "flops_per_step": flops / max(1, self.steps_timed),
                "contracted_points_per_assembly": (stats["timed_plastic_evals"] / max(1, stats["timed_assemblies"])
                                                   if not self.finite else cfg["K"]),
                "executed_dmma_tflops": executed / (kms / 1e3) / 1e12 if kms else None,
                "algorithmic_equiv": equiv,
                "avg_launch_ms": kms / launches_t, "share_of_step": kms / ms if ms else None}

    def roofline_hbm(self, stats, hbm, hbm_src):
        """DRAM traffic of the increment kernel: per launch every point reads its committed
        history (eps_p[4], eq: 40 B per J2 point) and writes its candidate (40 B) once; the
        repeated assembly passes of the Newton loop hit L2 (ncu: DRAM bytes per launch =
        1.02 x this, profiles/). achieved = that / the average launch time."""
        kms = stats["kernel_ms"]
        per_launch = self.P * self.model.K_j2 * 80.0
        gbs = per_launch * stats["timed_launches"] / (kms / 1e3) / 1e9 if kms else None
        return {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s",
                "frac": gbs / hbm if gbs else None, "peak_source": hbm_src,
                "kernel": "history stream of the increment kernel (eps_p[4], eq SoA, double-buffered)",
                "bytes_definition": "80 B per J2 cubature point per point per increment launch "
                                    "(40 B committed read + 40 B candidate write)",
                "bytes_per_launch": per_launch}


def mono_record(run, ms, its, st, P_total, peak, peak_src):
    """JSON record of a monolithic-scheme run (DeviceRun.mono_step)."""
    n_inc = len(its)
    pit = P_total * sum(its)
    rf = run.roofline(st, ms, peak, peak_src)
    rf["kernel"] = ("k_increment<..., MONO>" if run.cfg["n"] <= 32 else "k_increment_big<NT, MONO>") + \
        " (one condensed reduced-Newton iteration per launch)"
    return {"value": P_total * n_inc / (ms / 1e3), "unit": UNIT,
            "point_iterations_per_s": pit / (ms / 1e3), "iterations_per_increment": its,
            "ms_per_step": ms, "tol": 1e-8,
            "api": "per iteration: fe2_hrom_mono_iterate_device + fe2_hrom_gather (NCCL all-gather of "
                   "{Σ, C_macro, ‖r‖, status} + max all-reduce of failed / above-tol; lockstep termination); "
                   "fe2_hrom_mono_begin / _commit per increment",
            "exchanges": sum(its), "roofline": rf,
            "note": "evals/s = converged increments (all points below tol) per second, the unit of `value`"}


def main():
    args = parse()
    # the JSON line must be the only stdout line: keep NCCL's version banner off stdout
    if os.environ.get("NCCL_DEBUG", "VERSION").upper() == "VERSION":
        os.environ["NCCL_DEBUG"] = "WARN"
    cfg = dict(CONFIGS[args.config])
    if args.points:
        cfg["P"] = args.points
    if args.impl == "reference":
        run_reference(args, cfg)
        return

    import torch
    import torch.distributed as dist

    import paper_2306_02687_b200 as F

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
        # the engine's own NCCL communicator for the per-increment exchange
        uid = [F.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        COMM[0] = F.NcclComm(local, ws, rank, uid[0])
    # a dedicated stream (not the legacy default stream, whose handle 0 the C ABI reads as "the
    # engine's own stream"): torch's events, copies and the engine's kernels all run on it
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)

    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def timed(fn, steps):
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        barrier()
        ms = e0.elapsed_time(e1)
        if ws > 1:
            t = torch.tensor([ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    try:
        peak = json.load(open(DMMA_PEAK_FILE))["dmma_tflops_w16"]
        peak_src = "measured DMMA m8n8k4 f64 peak on this pool's B200 (tools/fp64_peak.cu, profiles/r01_fp64_peak.json)"
    except Exception:
        peak, peak_src = 37.0, "fallback: DMMA peak estimate"

    try:
        hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
        hbm_src = "MEASURED_PEAKS.json"
    except Exception:
        hbm, hbm_src = 6650.0, "fallback 6.65 TB/s"
    if COMM[0] is None and args.mono:  # one-rank communicator: the N = 1 exchange runs the same path
        COMM[0] = F.NcclComm(local, 1, 0, F.nccl_unique_id())

    run = DeviceRun(F, torch, cfg, rank, local, dev, stream, ws)
    eng, model, P, incr = run.eng, run.model, run.P, cfg["incr"]
    nc, nt = run.nc, run.nt
    for _ in range(args.warmup):
        run.device_step(dist, ws)
    run.check_converged()  # correctness guard on the warm-up trajectory

    eng.reset_stats()
    eng.set_timing(True)
    launches0 = eng.stats()["kernel_launches"]
    with ClockSampler(local) as clk:
        ms = timed(lambda: run.device_step(dist, ws), args.steps)
    stats = eng.stats()
    eng.set_timing(False)
    run.steps_timed = args.steps
    launches = stats["kernel_launches"] - launches0
    P_total = cfg["P"] if cfg.get("strong") else ws * P
    evals = P_total * incr * args.steps
    value = evals / (ms / 1e3)

    # ---- e2e through the host-buffer C-ABI (pinned host memory)
    pin = lambda a: torch.from_numpy(a).pin_memory().numpy()
    E_pin = pin(run.E_inc)
    o_sig, o_C, o_res = pin(np.empty((P, nc))), pin(np.empty((P, nt))), pin(np.empty(P))
    o_it, o_pc, o_st = (pin(np.empty(P, dtype=np.int32)) for _ in range(3))
    e2e_bufs = []
    if ws > 1:  # the engine's own device output buffers, gathered after each host-API call
        p_sig, p_C, p_it, p_pc, p_res, p_st = eng.output_ptrs()
        e_sig = wrap_dev(p_sig, (P, nc), "<f8", dev)
        e_C = wrap_dev(p_C, (P, nt), "<f8", dev)
        e_res = wrap_dev(p_res, (P,), "<f8", dev)
        e_st = wrap_dev(p_st, (P,), "<i4", dev)
        e2e_bufs.extend([e_sig, e_C, e_res, e_st])

    def e2e_step():
        eng.reset_points()
        if ws == 1:  # asynchronous host-buffer API: output copies overlap the next increment
            for k in range(incr):
                eng.solve_increment_async_into(E_pin[k], o_sig, o_C, o_it, o_pc, o_res, o_st)
            eng.wait()
            return
        for k in range(incr):
            eng.solve_increment_into(E_pin[k], o_sig, o_C, o_it, o_pc, o_res, o_st)
            run.gather(dist, ws, e_sig, e_C, e_res, e_st)

    e2e_step()
    e2e_steps = max(1, min(args.steps, 3))
    ms_e2e = timed(e2e_step, e2e_steps)
    e2e_value = P_total * incr * e2e_steps / (ms_e2e / 1e3)
    h2d = incr * P * nc * 8
    d2h = incr * P * (nc * 8 + nt * 8 + 8 + 3 * 4)

    # ---- the monolithic scheme (the paper's method) on the same workload: every macro
    # iteration advances each micro problem by ONE reduced Newton iteration and returns the
    # condensed Σ and C_macro; after EVERY iteration the records of all points are
    # all-gathered over NCCL (fe2_hrom_gather, also at N = 1 with a one-rank communicator)
    # and the ranks stop together when no point is above the tolerance.
    mono = None
    if args.mono and not run.finite:
        run.mono_step()
        run.eng.reset_stats()
        run.eng.set_timing(True)
        its_box = [None]
        ms_mono = timed(lambda: its_box.__setitem__(0, run.mono_step()), 1)
        mst = run.eng.stats()
        run.eng.set_timing(False)
        its = its_box[0]
        mono = mono_record(run, ms_mono, its, mst, P_total, peak, peak_src)

    # ---- the batched constitutive update on SoA HBM buffers (north_star item 1):
    # the HBM-bound kernel, timed alone on device-resident inputs: strains U[±0.03]
    # from a history with eq U[0, 0.01] (most points return plastically)
    constitutive = None
    if args.constitutive_points > 0:
        Nm = args.constitutive_points
        g = torch.Generator(device=dev).manual_seed(1234 + rank)
        c_eps = (torch.rand((3, Nm), dtype=torch.float64, device=dev, generator=g) - 0.5) * 0.06
        c_h = [torch.zeros((6, Nm), dtype=torch.float64, device=dev) for _ in range(2)]
        c_h[0][:4] = (torch.rand((4, Nm), dtype=torch.float64, device=dev, generator=g) - 0.5) * 0.004
        c_h[0][2] = -(c_h[0][0] + c_h[0][1])
        c_h[0][4] = torch.rand(Nm, dtype=torch.float64, device=dev, generator=g) * 0.01
        c_sig = torch.empty((3, Nm), dtype=torch.float64, device=dev)
        c_C6 = torch.empty((6, Nm), dtype=torch.float64, device=dev)
        c_pl = torch.empty(Nm, dtype=torch.uint8, device=dev)
        j2 = F.J2LinearParams()

        def mat_step(k):
            F.update_material_soa_device(j2, Nm, c_eps.data_ptr(), c_h[0].data_ptr(), c_sig.data_ptr(),
                                         c_C6.data_ptr(), c_h[1].data_ptr(), c_pl.data_ptr(),
                                         stream.cuda_stream, device=local)

        for k in range(3):
            mat_step(k)
        reps = 10
        cnt = [0]

        def mat_rep():
            mat_step(cnt[0])
            cnt[0] += 1

        mms = timed(lambda: [mat_rep() for _ in range(reps)], 1)
        # read eps (3) + history (5) = 64 B, write sigma (3) + C6 (6) + history (6) = 120 B + 1 B flag
        bpp = 64 + 120 + 1
        gbs = bpp * Nm * reps / (mms / 1e3) / 1e9
        try:
            hbm_pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
        except Exception:
            hbm_pk = 6650.0
        constitutive = {"bound": "hbm", "kernel": "k_material_soa (fe2_material_update_soa_device)",
                        "points": Nm, "launches": reps, "ms_per_launch": mms / reps,
                        "bytes_per_point": bpp, "achieved": gbs, "peak": hbm_pk, "unit": "GB/s",
                        "frac": gbs / hbm_pk, "evals_per_s": Nm * reps / (mms / 1e3),
                        "plastic_fraction": float(c_pl.float().mean().item())}
        del c_eps, c_h, c_sig, c_C6, c_pl

    # ---- other BASELINE configs, device-resident (same rank layout: weak for configs 1/2,
    # strong for config 3, whose points are split over the ranks)
    extras = {}
    for c in [int(x) for x in args.extra_configs.split(",") if x.strip()]:
        if c == 4 and ws == 1:  # the roofline sweep: a single-GPU experiment (BASELINE configs[4])
            extras["config4_roofline_sweep"] = config4_sweep()
            torch.cuda.set_stream(stream)  # run_cell works on a stream of its own
            continue
        if c == args.config or c not in CONFIGS:
            continue
        xcfg = dict(CONFIGS[c])
        xrun = DeviceRun(F, torch, xcfg, rank, local, dev, stream, ws)
        xrun.device_step(dist, ws, n_incr=2)  # warm-up: the first increments (kernels, allocations)
        xrun.eng.reset_stats()
        xrun.eng.set_timing(True)
        xms = timed(lambda: xrun.device_step(dist, ws), 1)
        xrun.check_converged()
        xst = xrun.eng.stats()
        xrun.eng.set_timing(False)
        xP_total = xcfg["P"] if xcfg.get("strong") else ws * xcfg["P"]
        xev = xP_total * xcfg["incr"]
        rec = {
            "value": xev / (xms / 1e3), "unit": UNIT, "steps": 1, "warmup": "2 increments", "ms_per_step": xms,
            "points_total": xP_total, "points_per_rank": xrun.P, "modes": xcfg["n"], "cubature": xcfg["K"],
            "cubature_j2": xrun.model.K_j2, "increments": xcfg["incr"],
            "scaling": "strong" if xcfg.get("strong") else "weak",
            "roofline": xrun.roofline(xst, xms, peak, peak_src),
            "newton": {"assemblies_per_eval": xst["timed_assemblies"] / (xrun.P * xcfg["incr"])},
            "parity": "unpinned (no reference finite-strain code; oracle fs_* checked by tests/test_gpu_fs.py)"
            if xrun.finite else "oracle parity tests/test_gpu_full_configs.py"}
        if not xrun.finite:
            rec["roofline_hbm"] = xrun.roofline_hbm(xst, hbm, hbm_src)
        nprof = os.path.join(ROOT, "profiles", "ncu_increment_summary.json")
        if os.path.exists(nprof):  # the kernel's ncu capture: pipe utilisation, DRAM bytes (scaled to P)
            try:
                e = json.load(open(nprof)).get(xcfg["name"], {})
                if e:
                    rec["roofline"]["ncu"] = {k: e.get(k) for k in ("dmma_pipe_pct_active", "fp64_pipe_pct_active",
                                                                    "issue_active_pct", "source")}
                    if e.get("dram_bytes_per_launch") and e.get("points"):
                        rec["roofline"]["traffic"] = e["dram_bytes_per_launch"] * xrun.P / e["points"]
            except Exception:
                pass
        if c == 3 and args.mono:  # the north_star multi-GPU scheme: exchange every Newton iteration
            xrun.eng.reset_stats()
            xrun.eng.set_timing(True)
            its_box = [None]
            mms = timed(lambda: its_box.__setitem__(0, xrun.mono_step()), 1)
            mst = xrun.eng.stats()
            xrun.eng.set_timing(False)
            rec["monolithic"] = mono_record(xrun, mms, its_box[0], mst, xP_total, peak, peak_src)
        extras[xcfg["name"]] = rec
        del xrun

    if rank != 0:
        COMM[0].close()
        dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel (one persistent launch per increment)
    roofline = run.roofline(stats, ms, peak, peak_src)
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_increment_summary.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get(cfg["name"], {}).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    roofline["traffic"] = traffic
    if os.path.exists(prof):  # the pipe utilisation of the same kernel from its ncu capture
        try:
            e = json.load(open(prof)).get(cfg["name"], {})
            roofline["ncu"] = {k: e.get(k) for k in ("dmma_pipe_pct_active", "fp64_pipe_pct_active",
                                                     "issue_active_pct", "warps_active_pct", "source")}
        except Exception:
            pass
    if constitutive is not None and os.path.exists(prof):
        try:
            constitutive["traffic"] = json.load(open(prof)).get("constitutive_soa", {}).get("dram_bytes_per_launch")
        except Exception:
            pass
    K_j2 = model.K_j2
    roofline_hbm = run.roofline_hbm(stats, hbm, hbm_src)
    if os.path.exists(prof):
        try:
            roofline_hbm["traffic"] = json.load(open(prof)).get(cfg["name"], {}).get("dram_bytes_per_launch")
        except Exception:
            pass

    cpu = None
    if not args.no_cpu_baseline and ws == 1:
        threads = os.cpu_count() or 1
        n_pts = args.cpu_sample_points or calibrate_cpu_points(cfg, threads, seconds=12.0)
        v, dt = cpu_reference_run(cfg, n_pts, threads)
        cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"first {n_pts} points x {incr} increments of {cfg['name']} ({dt:.1f} s)"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong" if cfg.get("strong") else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded Φ, cubature and paths, BASELINE configs)",
        "config": {"workload": cfg["name"], "points_per_rank": P, "modes": cfg["n"], "cubature": cfg["K"],
                   "cubature_j2": model.K_j2, "increments": incr, "parallelism": f"dp{ws} (points sharded)",
                   "l2": "inputs larger than L2 (history %.2f GB per rank > 126 MB L2)" % (P * model.K_j2 * 48 / 1e9),
                   "step": "one full trajectory of all points (reset to virgin state)"},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "steps": e2e_steps,
                "api": "fe2_hrom_solve_increment_async + fe2_hrom_wait (host buffers, pinned)" if ws == 1 else
                       "fe2_hrom_solve_increment (host buffers, pinned) + NCCL all-gather"},
        "gpu_launches": launches,
        "roofline": roofline,
        "roofline_hbm": roofline_hbm,
        "roofline_constitutive": constitutive,
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
        "newton": {"assemblies_per_eval": stats["timed_assemblies"] / (P * incr * args.steps),
                   "commits_per_eval": stats["timed_commits"] / (P * incr * args.steps),
                   "plastic_fraction": stats["timed_plastic_evals"] / max(1, stats["timed_assemblies"] * K_j2)},
        "extra_configs": extras,
        "monolithic": mono,
    }
    print(json.dumps(line), flush=True)
    if COMM[0] is not None:
        COMM[0].close()
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
