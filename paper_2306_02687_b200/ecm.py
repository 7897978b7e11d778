"""Offline hyper-integration rule by the Empirical Cubature Method (SURVEY
§8(f) rank 3): force snapshots from full-rule training
trajectories on the device engine, their SVD, and the ECM point selection
(fe2_ecm_select, host C++). Offline tooling around the online engine."""
from __future__ import annotations

import ctypes as C

import numpy as np

from .hrom import HyperRomEngine, HyperRomModel, _check, lib, make_paths

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
lib.fe2_ecm_select.argtypes = [_dp, _dp, C.c_int, C.c_int, C.c_int, C.c_double, _ip, _dp, _ip, _dp]


def ecm_select(U, w_full, m_target, tol=1e-6):
    """ECM on an integrand basis U (m x k) with full-rule weights w_full (m).
    Returns (point ids, positive weights, relative residual)."""
    U = np.ascontiguousarray(U, dtype=np.float64)
    w_full = np.ascontiguousarray(w_full, dtype=np.float64)
    m, k = U.shape
    cap = max(1, min(m_target, k + 1))
    ids, w = np.empty(cap, dtype=np.int32), np.empty(cap)
    n, res = C.c_int(), C.c_double()
    _check(lib.fe2_ecm_select(U.ctypes.data_as(_dp), w_full.ctypes.data_as(_dp), m, k, m_target, tol,
                              ids.ctypes.data_as(_ip), w.ctypes.data_as(_dp), C.byref(n), C.byref(res)))
    return ids[:n.value].copy(), w[:n.value].copy(), res.value


def force_snapshots(model: HyperRomModel, paths, engine: HyperRomEngine | None = None):
    """Integrand snapshots (collect_force_snapshots): for every (training
    point, converged increment) the per-integration-point values of the
    reduced-force integrand (G_q^T sigma_q)[a], a < n, and of the stress
    sigma_q (3) whose integral is the homogenised stress, on a FULL-rule
    model (K = all points). Columns of the returned (m x n_snap*(n+3))."""
    eng = engine or HyperRomEngine.from_model(model)
    P, incr, _ = paths.shape
    eng.alloc_points(P)
    lam = {}
    for mid, mat in enumerate(model.materials):  # Lamé parameters of each material
        lam[mid] = (mat.E * mat.nu / ((1 + mat.nu) * (1 - 2 * mat.nu)), mat.E / (2 * (1 + mat.nu)))
    G = model.G  # (K, 3, n)
    cols = []
    for k in range(incr):
        out = eng.solve_increment(paths[:, k])
        assert (out["status"] == 0).all()
        alpha, state, _ = eng.read_state()
        eps = paths[:, k][:, None, :] + np.einsum("qin,pn->pqi", G, alpha)  # (P, K, 3)
        ep = state[:, :, :4]
        lt = np.zeros(eps.shape[:2])
        sig = np.empty_like(eps)
        for mid, (la, mu) in lam.items():
            sel = model.mat == mid
            x0 = eps[:, sel, 0] - ep[:, sel, 0]
            x1 = eps[:, sel, 1] - ep[:, sel, 1]
            x2 = -ep[:, sel, 2]
            x3 = 0.5 * eps[:, sel, 2] - ep[:, sel, 3]
            lt = la * (x0 + x1 + x2)
            sig[:, sel, 0] = lt + 2 * mu * x0
            sig[:, sel, 1] = lt + 2 * mu * x1
            sig[:, sel, 2] = 2 * mu * x3
        f = np.einsum("qin,pqi->pqn", G, sig)  # (P, K, n) reduced-force integrand
        f = np.concatenate([f, sig], axis=2)  # + the homogenised-stress integrand (Σ = ∫σ / V)
        cols.append(f.transpose(1, 0, 2).reshape(model.K, -1))
    return np.concatenate(cols, axis=1)


def build_rule(model_full: HyperRomModel, paths, m_target, tol=1e-6, svd_tol=1e-10):
    """Training snapshots -> SVD -> ECM. Returns (ids, weights, residual, k modes)."""
    X = force_snapshots(model_full, paths)
    Uf, S, _ = np.linalg.svd(X, full_matrices=False)
    k = int(np.sum(S > svd_tol * S[0]))
    ids, w, res = ecm_select(Uf[:, :k], model_full.w, m_target, tol)
    return ids, w, res, k


def save_rule(path, ids, weights):
    """CubatureRule as text (SPEC.md hyper External Interfaces): one
    "point_id weight" line per point, weights in %.17g (bit-exact)."""
    with open(path, "w") as f:
        f.write(f"fe2rom-rule 1\n{len(ids)}\n")
        for q, w in zip(ids, weights):
            f.write(f"{int(q)} {float(w):.17g}\n")


def load_rule(path):
    with open(path) as f:
        head = f.readline().split()
        if head != ["fe2rom-rule", "1"]:
            raise ValueError("not a fe2rom rule file")
        m = int(f.readline())
        rows = [f.readline().split() for _ in range(m)]
    ids = np.array([int(r[0]) for r in rows], dtype=np.int32)
    w = np.array([float(r[1]) for r in rows])
    if (w <= 0).any() or len(set(ids.tolist())) != m:
        raise ValueError("rule weights must be positive and point ids unique")
    return ids, w
