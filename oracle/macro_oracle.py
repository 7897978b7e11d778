"""CPU ORACLE of the macro FE driver (test infrastructure only).

Restates, in numpy, the beam problem of fe2_macro_run (SPEC.md:455-518,
nested variant; build_beam_mesh mesh.hpp:133-169; shape_eval :85-115) on top
of the hyper-ROM oracle (pyoracle.Hrom). The oracle engine has no per-point
state API, so a micro solve "from the committed state" is a replay of the
committed macro strain path plus the trial strain from the virgin state —
the same increments (and bisections) the device engine runs after
fe2_hrom_restore.
"""
from __future__ import annotations

import numpy as np

import pyoracle as O

GP = np.array([[1.0 / 6.0, 1.0 / 6.0], [2.0 / 3.0, 1.0 / 6.0], [1.0 / 6.0, 2.0 / 3.0]])


def tri6_B(x, y, xi, eta):
    l1, l2, l3 = 1.0 - xi - eta, xi, eta
    g = np.array([[-(4 * l1 - 1), -(4 * l1 - 1)], [4 * l2 - 1, 0.0], [0.0, 4 * l3 - 1], [4 * (l1 - l2), -4 * l2],
                  [4 * l3, 4 * l2], [-4 * l3, 4 * (l1 - l3)]])
    J = np.array([[g[:, 0] @ x, g[:, 0] @ y], [g[:, 1] @ x, g[:, 1] @ y]])
    det = J[0, 0] * J[1, 1] - J[0, 1] * J[1, 0]
    Ji = np.array([[J[1, 1], -J[0, 1]], [-J[1, 0], J[0, 0]]]) / det
    dN = g @ Ji.T  # (6, 2): dN/dx, dN/dy
    B = np.zeros((3, 12))
    B[0, 0::2] = dN[:, 0]
    B[1, 1::2] = dN[:, 1]
    B[2, 0::2] = dN[:, 1]
    B[2, 1::2] = dN[:, 0]
    return B, det


def build_beam(L, H, nx, ny):
    gx, gy = 2 * nx + 1, 2 * ny + 1
    gid = lambda i, j: j * gx + i  # noqa: E731
    xy = np.array([[L * i / (gx - 1.0), H * j / (gy - 1.0)] for j in range(gy) for i in range(gx)])
    tri = []
    for j in range(ny):
        for i in range(nx):
            i0, j0 = 2 * i, 2 * j
            tri.append([gid(i0, j0), gid(i0 + 2, j0), gid(i0 + 2, j0 + 2), gid(i0 + 1, j0), gid(i0 + 2, j0 + 1),
                        gid(i0 + 1, j0 + 1)])
            tri.append([gid(i0, j0), gid(i0 + 2, j0 + 2), gid(i0, j0 + 2), gid(i0 + 1, j0 + 1),
                        gid(i0 + 1, j0 + 2), gid(i0, j0 + 1)])
    tri = np.array(tri)
    left = [gid(0, j) for j in range(gy)]
    tip = [gid(gx - 1, j) for j in range(gy)]
    B, w, elem = [], [], []
    for e, t in enumerate(tri):
        for xi, eta in GP:
            b, det = tri6_B(xy[t, 0], xy[t, 1], xi, eta)
            B.append(b)
            w.append(det / 6.0)
            elem.append(e)
    return dict(xy=xy, tri=tri, left=left, tip=tip, B=np.array(B), w=np.array(w), elem=np.array(elem))


class ReplayEngine:
    """Committed macro strain path + trial increment, replayed from the virgin state."""

    def __init__(self, hrom: O.Hrom, P, tol=1e-8, max_iter=30, max_bisections=4, threads=8):
        self.h, self.P = hrom, P
        self.opts = dict(tol=tol, max_iter=max_iter, max_bisections=max_bisections, threads=threads)
        self.path = []  # committed increments, each (P, 3)

    def solve(self, E):
        path = np.stack(self.path + [E], axis=1)  # (P, k, 3 | 4)
        r = self.h.run(path, **self.opts)
        fs = isinstance(self.h, O.HromFs)  # finite strain: P_M, A_M
        return dict(sigma=r["P" if fs else "sigma"][:, -1], C=r["A" if fs else "C"][:, -1], iters=r["iters"][:, -1],
                    status=r["status"][:, -1])

    def commit(self, E):
        self.path.append(np.array(E))


class MonoEngine:
    """Monolithic scheme: one reduced Newton iteration of
    every point per macro iteration, micro condensed (same algebra as
    fe2_hrom_mono_*): α -= K⁻¹(r + K_aE ΔE) with the previous iteration's
    factors, assemble at (E, α) from the committed history, return
    Σ~ = (Σ_raw − K_Eα K⁻¹ r)/V, C = (C_EE − K_Eα K⁻¹ K_aE)/V and |r|/ref with
    ref = max(|r| at the step's first iteration, |Σ_raw| now, 1e-30) — the
    current stress scale, since E itself moves during a monolithic step."""

    def __init__(self, hrom: O.Hrom, P, volume):
        self.h, self.P, self.V = hrom, P, volume
        n, K = hrom.n, hrom.K
        self.alpha_c = np.zeros((P, n))
        self.state_c = np.zeros((P, K, 6))
        self.first = True

    def begin(self):
        self.first = True

    def iterate(self, E):
        P, n, V = self.P, self.h.n, self.V
        if self.first:
            self.alpha_w = self.alpha_c.copy()
            self.ref = np.zeros(P)
        else:
            dE = E - self.E_w
            self.alpha_w = self.alpha_w - (self.zr + np.einsum("pai,pi->pa", self.Z, dE))
        self.zr, self.Z, self.E_w = np.zeros((P, n)), np.zeros((P, n, 3)), np.array(E, dtype=float)
        self.state_w = np.zeros_like(self.state_c)
        sig, Cm, rel, st = np.zeros((P, 3)), np.zeros((P, 3, 3)), np.zeros(P), np.zeros(P, dtype=int)
        for p in range(P):
            a = self.h.assemble(self.alpha_w[p], E[p], self.state_c[p])
            rn = np.linalg.norm(a["r"])
            if self.first:
                self.ref[p] = rn  # the step's initial micro residual
            ref = max(self.ref[p], np.linalg.norm(a["S_raw"]), 1e-30)
            try:
                L = np.linalg.cholesky(a["Kaa"])
            except np.linalg.LinAlgError:
                st[p] = 5
                continue
            solve = lambda b: np.linalg.solve(L.T, np.linalg.solve(L, b))  # noqa: E731
            self.zr[p] = solve(a["r"])
            self.Z[p] = solve(a["KaE"])
            q = a["KaE"].T @ self.Z[p]
            Cm[p] = (a["C_EE"] - 0.5 * (q + q.T)) / V
            sig[p] = (a["S_raw"] - a["KaE"].T @ self.zr[p]) / V
            rel[p] = rn / ref
            self.state_w[p] = a["state"]
        self.first = False
        return dict(sigma=sig, C=Cm, rel_res=rel, status=st)

    def commit(self):
        self.alpha_c = self.alpha_w.copy()
        self.state_c = self.state_w.copy()
        self.first = True


def solve_program(m, engine, L=4.0, H=1.0, nx=8, ny=2, u_max=0.3, n_load=10, max_unload=30,
                  tol=1e-6, max_iter=20, max_bisections=4, micro_tol=1e-8):
    """Same algorithm as fe2_macro_run. Returns rows (U, R, macro iters,
    cumulative micro iters) and U_residual."""
    beam = build_beam(L, H, nx, ny) if m is None else m
    B, w, elem, tri = beam["B"], beam["w"], beam["elem"], beam["tri"]
    if isinstance(engine.h, O.HromFs):  # total Lagrangian: H = F - I from the gradient operator
        Bg = np.zeros((len(w), 4, 12))
        Bg[:, 0, 0::2] = B[:, 0, 0::2]
        Bg[:, 1, 0::2] = B[:, 2, 0::2]
        Bg[:, 2, 1::2] = B[:, 2, 1::2]
        Bg[:, 3, 1::2] = B[:, 1, 1::2]
        B = Bg
    P = len(w)
    nd = 2 * len(beam["xy"])
    role = np.zeros(nd, dtype=int)
    for n_ in beam["left"]:
        role[2 * n_] = role[2 * n_ + 1] = 1
    for n_ in beam["tip"]:
        role[2 * n_ + 1] = 2
    free = np.where(role == 0)[0]
    edofs = np.array([[2 * t[d // 2] + d % 2 for d in range(12)] for t in tri])
    gdofs = edofs[elem]  # (P, 12)
    u = np.zeros(nd)
    state = dict(micro=0, fint=np.zeros(nd), E=None, fscale=0.0, micro_ok=True)

    mono = isinstance(engine, MonoEngine)

    def micro_solve():
        E = np.einsum("gid,gd->gi", B, u[gdofs])
        if mono:
            out = engine.iterate(E)
            if (out["status"] != 0).any():
                return None
            state["micro"] += P
            state["micro_ok"] = bool((out["rel_res"] <= micro_tol).all())
        else:
            out = engine.solve(E)
            if (out["status"] != 0).any():
                return None
            state["micro"] += int(out["iters"].sum())
        fint = np.zeros(nd)
        np.add.at(fint, gdofs, w[:, None] * np.einsum("gid,gi->gd", B, out["sigma"]))
        state["fint"], state["E"] = fint, E
        return out

    def Kff_of(C):
        CB = np.einsum("gij,gjd->gid", C, B)
        Ke = w[:, None, None] * np.einsum("gia,gib->gab", B, CB)
        K = np.zeros((nd, nd))
        np.add.at(K, (gdofs[:, :, None], gdofs[:, None, :]), Ke)
        return K

    def predict(U):
        """Δu_f = -K_ff⁻¹ K_fp ΔU with the last accepted state's tangent."""
        dU = U - u[2 * beam["tip"][0] + 1]
        if dU == 0.0:
            return
        du = np.zeros(nd)
        for n_ in beam["tip"]:
            du[2 * n_ + 1] = dU
        K = Kff_of(state["C_acc"])
        u[free] += np.linalg.solve(K[np.ix_(free, free)], -(K @ du)[free])

    def macro_step(U):
        predict(U)
        for n_ in beam["tip"]:
            u[2 * n_ + 1] = U
        if mono:
            engine.begin()
        for k in range(max_iter + 1):
            out = micro_solve()
            if out is None:
                return -1
            fint = state["fint"]
            rn, fn = np.linalg.norm(fint[free]), np.linalg.norm(fint)
            state["C"] = out["C"]
            if rn <= tol * max(fn, state["fscale"], 1e-30) and (not mono or state["micro_ok"]):
                return k
            if k == max_iter:
                return -1
            state["C"] = out["C"]
            Kff = Kff_of(out["C"])[np.ix_(free, free)]
            u[free] += np.linalg.solve(Kff, -fint[free])
        return -1

    # tangent of the virgin state for the first step's predictor
    if mono:
        engine.begin()
    state["C_acc"] = micro_solve()["C"]
    state["micro"] = 0
    rows = []
    done_state = dict(U=0.0, u=u.copy())

    def advance(U_target):
        frac, bis, done, iters = 1.0, 0, 0.0, 0
        U0 = done_state["U"]
        while done < 1.0 - 1e-12:
            target = min(1.0, done + frac)
            U = U0 + (U_target - U0) * target
            k = macro_step(U)
            if k < 0:
                u[:] = done_state["u"]
                bis += 1
                if bis > max_bisections:
                    raise RuntimeError("macro step did not converge")
                frac *= 0.5
                continue
            iters += k
            if mono:
                engine.commit()
            else:
                engine.commit(state["E"])
            state["fscale"] = max(state["fscale"], np.linalg.norm(state["fint"]))
            done_state["U"], done_state["u"] = U, u.copy()
            state["C_acc"] = state["C"]
            done = target
        R = sum(state["fint"][2 * n_ + 1] for n_ in beam["tip"])
        rows.append((done_state["U"], R, iters, state["micro"]))

    dU = u_max / n_load
    for k in range(1, n_load + 1):
        advance(dU * k)
    ures = float("nan")
    for _ in range(max_unload):
        U_prev, R_prev = rows[-1][0], rows[-1][1]
        advance(done_state["U"] - dU)
        U, R = rows[-1][0], rows[-1][1]
        if (R_prev > 0) != (R > 0):
            ures = U_prev + (U - U_prev) * (R_prev / (R_prev - R))
            break
    return np.array(rows), ures
