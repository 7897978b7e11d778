"""Macro FE driver of the two-scale beam over the native C ABI
(fe2_macro_*; SPEC.md:455-518 fe2.macro_step / solve_program, nested
variant). The macro loop is host C++ in the library;
every macro Newton iteration is one engine increment for all macro Gauss
points on the device (nested), or one monolithic micro iteration of all of
them (scheme="monolithic": fe2_hrom_mono_*)."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from .hrom import HyperRomEngine, NewtonOptions, _check, _Opts, lib


class _MacroCfg(C.Structure):
    _fields_ = [("length", C.c_double), ("height", C.c_double), ("nx", C.c_int), ("ny", C.c_int),
                ("u_max", C.c_double), ("n_load", C.c_int), ("max_unload", C.c_int), ("tol", C.c_double),
                ("max_iter", C.c_int), ("max_bisections", C.c_int), ("micro", _Opts), ("scheme", C.c_int)]


lib.fe2_macro_points.argtypes = [C.POINTER(_MacroCfg), C.POINTER(C.c_int64)]
lib.fe2_macro_gauss.argtypes = [C.POINTER(_MacroCfg), C.POINTER(C.c_double), C.POINTER(C.c_double),
                                C.POINTER(C.c_int)]
lib.fe2_macro_run.argtypes = [C.POINTER(_MacroCfg), C.c_void_p, C.POINTER(C.c_double), C.c_int,
                              C.POINTER(C.c_int), C.POINTER(C.c_double)]
lib.fe2_macro_run_hf.argtypes = lib.fe2_macro_run.argtypes


@dataclass
class MacroConfig:
    """Desk beam (SPEC fe2 DESIGN DECISIONS): L/H = 4, 32 Tri6 elements."""
    length: float = 4.0
    height: float = 1.0
    nx: int = 8
    ny: int = 2
    u_max: float = 0.3
    n_load: int = 10
    max_unload: int = 30
    tol: float = 1e-6
    max_iter: int = 20
    max_bisections: int = 4
    micro: NewtonOptions = field(default_factory=NewtonOptions)
    scheme: str = "nested"  # or "monolithic"

    def _c(self):
        assert self.scheme in ("nested", "monolithic")
        return _MacroCfg(self.length, self.height, self.nx, self.ny, self.u_max, self.n_load, self.max_unload,
                         self.tol, self.max_iter, self.max_bisections, self.micro._c(),
                         1 if self.scheme == "monolithic" else 0)


def macro_points(cfg: MacroConfig) -> int:
    n = C.c_int64()
    _check(lib.fe2_macro_points(C.byref(cfg._c()), C.byref(n)))
    return n.value


def macro_gauss(cfg: MacroConfig):
    """Per macro Gauss point: B (3 x 12), weight, element."""
    P = macro_points(cfg)
    B, w, e = np.empty((P, 3, 12)), np.empty(P), np.empty(P, dtype=np.int32)
    _check(lib.fe2_macro_gauss(C.byref(cfg._c()), B.ctypes.data_as(C.POINTER(C.c_double)),
                               w.ctypes.data_as(C.POINTER(C.c_double)), e.ctypes.data_as(C.POINTER(C.c_int))))
    return B, w, e


def solve_program(cfg: MacroConfig, engine, max_rows: int = 256):
    """Load / unload program on the beam (solve_program). engine: a
    HyperRomEngine (hyper-ROM FE²; the plain ROM is a full-rule model, K = 0)
    or a pod.HfRve (full-field HF FE²) — the four methods of SPEC.md:461 with
    cfg.scheme nested or monolithic on either. Returns the curve rows (U, R, macro iterations, cumulative micro
    iterations, wall ms) and the residual displacement U_res of the unloaded beam."""
    P = macro_points(cfg)
    if getattr(engine, "P", 0) != P:
        engine.alloc_points(P)
    rows = np.empty((max_rows, 5))
    n, ures = C.c_int(), C.c_double()
    run = lib.fe2_macro_run if isinstance(engine, HyperRomEngine) else lib.fe2_macro_run_hf
    _check(run(C.byref(cfg._c()), engine._h, rows.ctypes.data_as(C.POINTER(C.c_double)), max_rows, C.byref(n),
               C.byref(ures)))
    r = rows[:n.value]
    return dict(U=r[:, 0].copy(), R=r[:, 1].copy(), macro_iters=r[:, 2].astype(int),
                micro_iters=r[:, 3].astype(np.int64), wall_ms=r[:, 4].copy(), U_residual=ures.value)


def curve_error(test, ref):
    """curve_error: max over the common U grid of
    |R_test - R_ref| / max |R_ref|, both curves interpolated linearly on the
    load branch (rows up to the peak U)."""
    def branch(c):
        k = int(np.argmax(c["U"])) + 1
        return c["U"][:k], c["R"][:k]
    Ut, Rt = branch(test)
    Ur, Rr = branch(ref)
    lo, hi = max(Ut[0], Ur[0]), min(Ut[-1], Ur[-1])
    if not hi > lo:
        raise ValueError("curves do not overlap")
    grid = np.union1d(Ut[(Ut >= lo) & (Ut <= hi)], Ur[(Ur >= lo) & (Ur <= hi)])
    return float(np.abs(np.interp(grid, Ut, Rt) - np.interp(grid, Ur, Rr)).max() / np.abs(Rr).max())
