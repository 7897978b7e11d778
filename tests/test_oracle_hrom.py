"""The oracle's hyper-ROM online path (the restatement the GPU is checked
against): the SPEC.md:591 bridge to the HF restatement, condensation and
Newton semantics, determinism."""
import numpy as np
import pytest

import pyoracle as O

DESK = [("j2", 1.0, 0.3, 0.01, 0.016), ("elastic", 10.0, 0.3)]


def test_full_basis_full_rule_equals_hf():
    """SPEC.md:591 oracle equivalence: Φ = identity on the free DOFs and the
    full quadrature reproduce the HF micro solve (micro_newton + homogenize)."""
    mesh = O.Mesh(0, 6)
    md = O.Model(n=0, K=0, seed=0, mesh=mesh)
    assert md.n == md.n_free and md.K == 3 * mesh.n_elements
    path = np.array([[0.005, -0.002, 0.003], [0.01, -0.004, 0.006], [0.02, -0.008, 0.012], [0.01, -0.004, 0.006]])
    hf = mesh.hf_trajectory(DESK, path, tol=1e-12)
    hr = O.Hrom(md.G, md.w, md.mat, DESK, md.volume).run(path[None], tol=1e-12)
    assert (hr["status"] == 0).all()
    for k in range(len(path)):
        s, C = hr["sigma"][0, k], hr["C"][0, k]
        assert np.linalg.norm(s - hf["sigma"][k]) < 1e-9 * np.linalg.norm(hf["sigma"][k])
        assert np.abs(C - hf["C"][k]).max() < 1e-9 * np.abs(hf["C"][k]).max()
    assert hr["plastic_count"][0].max() > 0


def test_homogeneous_bridge_exact():
    """test_rve.cpp:44-62 through the reduced path: zero fluctuation, C = C_e."""
    mesh = O.Mesh(geometry=1, subdivisions=4)
    md = O.Model(n=0, K=0, seed=0, mesh=mesh)
    E = np.array([[[0.01, -0.004, 0.006]]])
    r = O.Hrom(md.G, md.w, md.mat, [("elastic", 2.0, 0.25)], md.volume).run(E, final_state=True)
    lam, mu = 2.0 * 0.25 / (1.25 * 0.5), 1.0 / 1.25
    Ce = np.array([[lam + 2 * mu, lam, 0], [lam, lam + 2 * mu, 0], [0, 0, mu]])
    assert r["iters"][0, 0] <= 1
    assert np.abs(r["alpha"]).max() < 1e-10
    np.testing.assert_allclose(r["C"][0, 0], Ce, atol=1e-8 * Ce.max())


def small_model():
    md = O.Model(8, 8, 60, 3)
    return md, O.Hrom(md.G, md.w, md.mat, DESK, md.volume)


def test_reduced_condensed_tangent_matches_fd():
    """The condensation C = (C_EE - K_Ea K_aa^-1 K_aE)/V is the exact
    derivative of the converged macro stress (cf. test_rve.cpp:163-195)."""
    md, h = small_model()
    for E in (np.array([0.004, -0.001, 0.002]), np.array([0.03, -0.01, 0.02])):
        r = h.run(E[None, None], tol=1e-13)
        C = r["C"][0, 0]
        fd = np.zeros((3, 3))
        for j in range(3):
            ep, em = E.copy(), E.copy()
            ep[j] += 1e-7
            em[j] -= 1e-7
            fd[:, j] = (h.run(ep[None, None], tol=1e-13)["sigma"][0, 0] - h.run(em[None, None], tol=1e-13)["sigma"][0, 0]) / 2e-7
        assert np.abs(C - fd).max() < 1e-5 * np.abs(C).max()
        assert np.abs(C - C.T).max() < 1e-12 * np.abs(C).max()
        assert np.linalg.eigvalsh(0.5 * (C + C.T)).min() > 0


def test_newton_iteration_semantics():
    """micro_newton counting (rve.hpp:300-315): a linear (elastic) increment
    converges after one step, re-solving the converged state needs none."""
    md, h = small_model()
    E = np.array([1e-4, -2e-5, 5e-5])
    r = h.run(np.stack([E, E])[None])
    assert list(r["iters"][0]) == [1, 0]
    assert list(r["plastic_count"][0]) == [0, 0]


def test_deterministic_and_thread_independent():
    md = O.Model(33, 12, 200, 0)
    E = O.paths(0, 0, 12, 6)
    h = O.Hrom(md.G, md.w, md.mat, DESK, md.volume)
    a = h.run(E, threads=1)
    b = h.run(E, threads=4)
    for k in ("sigma", "C", "iters", "plastic_count", "res_norm"):
        assert np.array_equal(a[k], b[k]), k


def test_bisection_path_is_exercised():
    """run_trajectory bisection (rve.hpp:473-478): with max_iter = 2 a large
    plastic increment fails, is halved, and the sub-steps converge; with
    max_iter = 1 it exhausts the bisections (ErrorCode::solver)."""
    md, h = small_model()
    E = np.array([[[0.03, -0.01, 0.02]]])
    r = h.run(E, max_iter=2, max_bisections=8)
    assert r["status"][0, 0] == 0 and r["bisections"][0, 0] >= 1
    ref = h.run(E)
    assert np.linalg.norm(r["sigma"] - ref["sigma"]) < 5e-2 * np.linalg.norm(ref["sigma"])
    r = h.run(E, max_iter=1, max_bisections=3)
    assert r["status"][0, 0] == 5  # 1 + ErrorCode::solver
    assert np.isnan(r["sigma"][0, 0]).all()
