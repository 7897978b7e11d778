"""Finite-strain (Biot stress) oracle, BASELINE config 2 — PARITY UNPINNED.

The reference has no finite-strain code, so the
oracle is anchored by properties instead of golden vectors: the consistent
tangent against central differences (the pattern of test_materials.cpp:210-271),
objectivity, the small-strain limit back to the PINNED small-strain material
and hyper-ROM oracle, and the 4-row operator against the pinned 3-row G_q.
"""
import numpy as np
import pytest

import pyoracle as O

J2 = ("j2", 1.0, 0.3, 0.01, 0.016)
EL = ("elastic", 10.0, 0.3)
DESK = [J2, EL]
M = np.array([[1, 0, 0, 0], [0, 0, 0, 1], [0, 1, 1, 0]], dtype=float)  # H -> (e11, e22, g12)


def _rot(th):
    return np.array([[np.cos(th), -np.sin(th)], [np.sin(th), np.cos(th)]])


def _fd_A(mat, state, F, h=1e-7):
    A = np.zeros((4, 4))
    for k in range(4):
        fp, fm = F.copy(), F.copy()
        fp[k] += h
        fm[k] -= h
        A[:, k] = (O.update_biot(mat, state, fp)[0] - O.update_biot(mat, state, fm)[0]) / (2 * h)
    return A


def _random_F(rng, amp=0.06):
    while True:
        H = rng.uniform(-amp, amp, 4)
        if (1 + H[0]) * (1 + H[3]) - H[1] * H[2] > 0.8:
            return np.array([1.0, 0.0, 0.0, 1.0]) + H


@pytest.mark.parametrize("mat", [J2, EL])
def test_biot_tangent_matches_central_differences(mat):
    rng = np.random.default_rng(3)
    n_plastic = 0
    for _ in range(20):
        # history from a previous (possibly plastic) step, then a fresh step
        _, _, st, _ = O.update_biot(mat, None, _random_F(rng))
        F = _random_F(rng)
        P, A, _, pl = O.update_biot(mat, st, F)
        n_plastic += pl
        fd = _fd_A(mat, st, F)
        assert np.abs(A - fd).max() <= 1e-6 * np.abs(A).max()
    if mat is J2:
        assert n_plastic > 5


def test_biot_objectivity():
    rng = np.random.default_rng(5)
    for _ in range(10):
        F = _random_F(rng)
        _, _, st, _ = O.update_biot(J2, None, _random_F(rng))
        P, A, so, pl = O.update_biot(J2, st, F)
        Q = _rot(rng.uniform(-np.pi, np.pi))
        P2, A2, so2, pl2 = O.update_biot(J2, st, (Q @ F.reshape(2, 2)).ravel())
        np.testing.assert_allclose(P2.reshape(2, 2), Q @ P.reshape(2, 2), atol=1e-14)
        np.testing.assert_allclose(so2, so, atol=1e-14)
        assert pl == pl2
        # dP/dF transforms as Q (A : Q^T dF)
        for k in range(4):
            dF = np.zeros(4)
            dF[k] = 1.0
            lhs = (A2 @ dF).reshape(2, 2)
            rhs = Q @ (A @ (Q.T @ dF.reshape(2, 2)).ravel()).reshape(2, 2)
            np.testing.assert_allclose(lhs, rhs, atol=1e-12)


def test_biot_pure_rotation_is_stress_free():
    for th in (0.1, 0.7, -2.0):
        P, _, so, pl = O.update_biot(J2, None, _rot(th).ravel())
        assert np.abs(P).max() < 1e-14 and not pl and np.abs(so[:5]).max() == 0.0


@pytest.mark.parametrize("mat", [J2, EL])
def test_biot_small_strain_limit(mat):
    """F = I + tH, t -> 0: P -> sigma(eps = sym H) of the pinned small-strain update."""
    rng = np.random.default_rng(7)
    H = rng.uniform(-1, 1, 4)
    for t in (1e-3, 1e-4):
        P, A, _, _ = O.update_biot(mat, None, np.array([1.0, 0, 0, 1.0]) + t * H)
        s, Cm, _, _ = O.update_material(mat, None, t * (M @ H))
        ref = np.array([s[0], s[2], s[2], s[1]])
        assert np.abs(P - ref).max() <= 5 * t * np.abs(ref).max()
    # at F = I the tangent is the small-strain one mapped to gradient components
    _, A, _, _ = O.update_biot(mat, None, np.array([1.0, 0, 0, 1.0]))
    _, Cm, _, _ = O.update_material(mat, None, np.zeros(3))
    Cg = Cm @ M
    np.testing.assert_allclose(A, np.array([Cg[0], Cg[2], Cg[2], Cg[1]]), atol=1e-14)


def test_g4_symmetric_part_is_pinned_g():
    md = O.Model(subdivisions=12, n=10, K=80, seed=4)
    G4 = O.model_g4(12, 10, 80, 4)
    np.testing.assert_array_equal(G4[:, 0], md.G[:, 0])
    np.testing.assert_array_equal(G4[:, 3], md.G[:, 1])
    np.testing.assert_allclose(G4[:, 1] + G4[:, 2], md.G[:, 2], atol=1e-15 * np.abs(md.G).max())


def test_paths_fs_shape_and_constraint():
    H = O.paths_fs(11, 500, 30)
    Hend = H[:, -1]
    assert np.abs(Hend).max() <= 0.08
    det = (1 + Hend[:, 0]) * (1 + Hend[:, 3]) - Hend[:, 1] * Hend[:, 2]
    assert (det > 0.8).all()
    k = np.arange(1, 31) / 30.0
    np.testing.assert_allclose(H, Hend[:, None, :] * k[None, :, None], rtol=1e-15, atol=0)
    np.testing.assert_array_equal(O.paths_fs(11, 5, 30, p0=100), H[100:105])


def _fs_model(n=8, K=60, sub=12, seed=1):
    md = O.Model(subdivisions=sub, n=n, K=K, seed=seed)
    G4 = O.model_g4(sub, n, K, seed)
    return md, O.HromFs(G4, md.w, md.mat, DESK, md.volume)


def test_fs_assembly_blocks_are_derivatives():
    md, h = _fs_model()
    rng = np.random.default_rng(2)
    # a plastic history state from a converged increment
    H0 = np.array([0.03, 0.02, -0.01, -0.02])
    run = h.run(H0[None, None, :], final_state=True)
    assert run["status"][0, 0] == 0
    st = run["state"][0]
    assert np.abs(st[:, 4]).max() > 0
    alpha = run["alpha"][0] + rng.normal(0, 0.01, h.n)
    H = H0[[0, 2, 1, 3]] * 1.2  # a non-coaxial next step from the plastic history
    A = h.assemble(alpha, H, st)
    eps = 1e-7
    Kfd, KaFfd, KFafd, CFFfd = (np.zeros_like(A["Kaa"]), np.zeros_like(A["KaF"]), np.zeros_like(A["KFa"]),
                                np.zeros_like(A["C_FF"]))
    for b in range(h.n):
        d = np.zeros(h.n)
        d[b] = eps
        ap, am = h.assemble(alpha + d, H, st), h.assemble(alpha - d, H, st)
        Kfd[:, b] = (ap["r"] - am["r"]) / (2 * eps)
        KFafd[:, b] = (ap["P_raw"] - am["P_raw"]) / (2 * eps)
    for s in range(4):
        d = np.zeros(4)
        d[s] = eps
        ap, am = h.assemble(alpha, H + d, st), h.assemble(alpha, H - d, st)
        KaFfd[:, s] = (ap["r"] - am["r"]) / (2 * eps)
        CFFfd[:, s] = (ap["P_raw"] - am["P_raw"]) / (2 * eps)
    assert A["plastic_count"] > 0
    for got, fd in ((A["Kaa"], Kfd), (A["KaF"], KaFfd), (A["KFa"], KFafd), (A["C_FF"], CFFfd)):
        assert np.abs(got - fd).max() <= 1e-5 * np.abs(got).max()
    # plastic flow not coaxial with the stretch: K_aa is not symmetric (-> LU)
    assert np.abs(A["Kaa"] - A["Kaa"].T).max() > 1e-6 * np.abs(A["Kaa"]).max()


def test_fs_condensed_tangent_matches_fd_of_macro_stress():
    _, h = _fs_model()
    H = np.array([0.004, -0.002, 0.001, 0.003])  # one elastic increment from the virgin state
    base = h.run(H[None, None, :], tol=1e-13)
    A = base["A"][0, 0]
    eps = 1e-7
    fd = np.zeros((4, 4))
    for s in range(4):
        d = np.zeros(4)
        d[s] = eps
        rp = h.run((H + d)[None, None, :], tol=1e-13)["P"][0, 0]
        rm = h.run((H - d)[None, None, :], tol=1e-13)["P"][0, 0]
        fd[:, s] = (rp - rm) / (2 * eps)
    assert base["plastic_count"][0, 0] == 0
    assert np.abs(A - fd).max() <= 1e-5 * np.abs(A).max()


def test_fs_small_strain_limit_of_reduced_path():
    """Small H: the finite-strain hyper-ROM reproduces the pinned small-strain
    hyper-ROM (Sigma, C) to O(|H|). (|H| is kept at 1e-4: U - I is formed by
    cancellation, so the finite-strain residual floor is ~1e-16 absolute.)"""
    md, h = _fs_model()
    Hs = 1e-4 * np.array([0.5, 0.3, -0.2, -0.4])
    fs = h.run(Hs[None, None, :])
    ss = O.Hrom(md.G, md.w, md.mat, DESK, md.volume).run((M @ Hs)[None, None, :])
    assert fs["status"][0, 0] == 0 and fs["plastic_count"][0, 0] == 0
    s, Cm = ss["sigma"][0, 0], ss["C"][0, 0]
    P, A = fs["P"][0, 0], fs["A"][0, 0]
    ref = np.array([s[0], s[2], s[2], s[1]])
    assert np.abs(P - ref).max() <= 1e-3 * np.abs(ref).max()
    Cg = Cm @ M
    np.testing.assert_allclose(A, np.array([Cg[0], Cg[2], Cg[2], Cg[1]]), atol=1e-3 * np.abs(Cg).max())


def test_fs_trajectory_converges_and_is_deterministic():
    _, h = _fs_model()
    H = O.paths_fs(0, 12, 10)
    r1 = h.run(H, threads=1)
    r4 = h.run(H, threads=4)
    assert (r1["status"] == 0).all()
    assert r1["plastic_count"].max() > 0
    assert (r1["iters"] >= 1).all()
    for k in ("P", "A", "iters", "plastic_count", "res_norm"):
        np.testing.assert_array_equal(r1[k], r4[k])


def test_fs_bisection_and_failure():
    _, h = _fs_model()
    H = O.paths_fs(0, 6, 2) * 1.0
    r = h.run(H, max_iter=2, max_bisections=8)
    assert (r["bisections"] > 0).any()
    f = h.run(H, max_iter=1, max_bisections=0)
    bad = f["status"] != 0
    assert bad.any()
    assert np.isnan(f["P"][bad]).all() and np.isnan(f["A"][bad]).all()


def test_biot_rotational_balance_measured():
    """Rotational balance: τ = P Fᵀ = R T U Rᵀ is symmetric iff T and U commute.
    MEASURED PROPERTY of this (parity-unpinned) formulation: exact
    (rounding) for elastic states and for a return from a history coaxial with U
    — the radial return keeps T coaxial with the trial deviator — but a plastic
    history εp that is not coaxial with the current stretch makes T non-coaxial
    and τ slightly unsymmetric (skew / |τ| up to ~1.4%, median 0.08%, at random
    |H| <= 0.06 and |εp| <= 0.01). The small-strain limit is unaffected."""
    rng = np.random.default_rng(0)

    def skew(P, F):
        t = P.reshape(2, 2) @ F.reshape(2, 2).T
        return abs(t[0, 1] - t[1, 0]) / np.linalg.norm(t)

    virgin, hist = [], []
    for _ in range(500):
        F = _random_F(rng)
        P, _, _, _ = O.update_biot(J2, np.zeros(6), F)
        virgin.append(skew(P, F))
        ep = rng.uniform(-0.01, 0.01, 4)
        ep[2] = -(ep[0] + ep[1])
        st = np.concatenate([ep, [rng.uniform(0.0, 0.02)], [0.0]])
        P, _, _, _ = O.update_biot(J2, st, F)
        hist.append(skew(P, F))
    assert max(virgin) < 1e-14
    assert 1e-4 < np.median(hist) < 5e-3 and max(hist) < 0.03
