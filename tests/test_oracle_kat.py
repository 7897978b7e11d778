"""Pin the CPU oracle to the reference's own known-answer tests.

Each test restates a Catch2 case of /root/reference/proj/tests (file:line in
the docstring) against the oracle's restatement of materials.hpp / rve.hpp.
"""
import numpy as np
import pytest

import pyoracle as O

J2 = ("j2", 1.0, 0.3, 0.01, 0.016)  # J2LinearParams defaults (materials.hpp:45-49)


def elastic_C(E, nu):
    lam = E * nu / ((1 + nu) * (1 - 2 * nu))
    mu = 0.5 * E / (1 + nu)
    return np.array([[lam + 2 * mu, lam, 0], [lam, lam + 2 * mu, 0], [0, 0, mu]])


def test_rng_is_mt19937_64():
    """common.hpp:56-88 — std::mt19937_64; the C++ standard's check value."""
    r = O.Rng(5489)
    for _ in range(9999):
        r.next_u64()
    assert r.next_u64() == 9981545732273789042
    r = O.Rng(42)
    u = [r.uniform() for _ in range(1000)]
    assert min(u) >= 0.0 and max(u) < 1.0
    ints = [r.uniform_int(7) for _ in range(2000)]
    assert min(ints) == 0 and max(ints) == 6
    n = np.array([r.normal() for _ in range(20000)])
    assert abs(n.mean()) < 0.03 and abs(n.std() - 1) < 0.03


def test_plane_strain_elasticity_closed_forms():
    """test_materials.cpp:49-69"""
    s, C, _, _ = O.update_material(("elastic", 1.0, 0.3), None, np.zeros(3))
    assert np.linalg.norm(s) == 0.0
    assert np.abs(C - C.T).max() < 1e-14
    assert np.linalg.eigvalsh(C).min() > 0.0
    s, C, _, _ = O.update_material(("elastic", 1.0, 0.0), None, np.array([1.0, 0, 0]))
    assert s[0] == pytest.approx(1.0, rel=1e-14) and abs(s[1]) < 1e-14 and abs(s[2]) < 1e-14
    E, nu = 1.0, 0.3
    s, C, _, _ = O.update_material(("elastic", E, nu), None, np.array([0.01, 0, 0]))
    assert s[0] == pytest.approx(E * (1 - nu) / ((1 + nu) * (1 - 2 * nu)) * 0.01, rel=1e-14)
    np.testing.assert_allclose(C, elastic_C(E, nu), rtol=1e-15)


def test_j2_elastic_step_leaves_state_untouched():
    """test_materials.cpp:71-78"""
    s, C, st, pl = O.update_material(J2, None, np.array([0.005, 0, 0]))
    assert st[4] == 0.0 and np.linalg.norm(st[:4]) == 0.0 and not pl
    assert np.abs(C - elastic_C(1.0, 0.3)).max() < 1e-14


def vonmises4(sig4):
    p = sig4[:3].sum() / 3.0
    d = np.array([sig4[0] - p, sig4[1] - p, sig4[2] - p, sig4[3]])
    return np.sqrt(1.5) * np.sqrt(d[0] ** 2 + d[1] ** 2 + d[2] ** 2 + 2 * d[3] ** 2)


def test_j2_uniaxial_strain_follows_hardening_line():
    """test_materials.cpp:80-101"""
    mu = 0.5 / 1.3
    st = np.zeros(6)
    for k in range(1, 26):
        e = 0.05 * k / 25
        s, C, st, _ = O.update_material(J2, st, np.array([e, 0, 0]))
        q = vonmises4(np.array([s[0], s[1], st[5], s[2]]))
        if st[4] > 0:
            assert abs(q - (0.01 + 0.016 * st[4])) < 1e-10 * 0.01
            eq_exact = (2 * mu * e - 0.01) / (3 * mu + 0.016)
            assert st[4] == pytest.approx(eq_exact, rel=1e-8)
        assert abs(st[0] + st[1] + st[2]) < 1e-10
    assert st[4] > 0


def test_j2_reversal_unloads_elastically():
    """test_materials.cpp:103-118"""
    e1 = np.array([0.017, 0.0, 0.002])
    s1, _, st1, pl = O.update_material(J2, None, e1)
    assert st1[4] > 0 and pl
    s2, _, st2, pl2 = O.update_material(J2, st1, np.zeros(3))
    assert not pl2
    assert np.linalg.norm(st2[:4]) == pytest.approx(np.linalg.norm(st1[:4]), rel=1e-12)
    expected = s1 - elastic_C(1.0, 0.3) @ e1
    assert np.linalg.norm(s2 - expected) < 1e-12
    assert np.linalg.norm(s2) > 1e-4


@pytest.mark.parametrize("name,mat", [("elastic", ("elastic", 1.0, 0.3)), ("j2", J2)])
def test_consistent_tangent_matches_central_fd(name, mat):
    """test_materials.cpp:210-271 — 120 random states from Rng(42), rel < 1e-6,
    plus the flow invariants (deviatoric flow, eq monotone, dissipation >= 0)."""
    rng = O.Rng(42)
    tested = guard = 0
    mu = 0.5 / 1.3
    while tested < 120 and guard < 5000:
        guard += 1
        st = np.zeros(6)
        eps = np.zeros(3)
        rng.uniform()  # dt = 0.5 + uniform() (rate independent here, consumed as the reference does)
        pre = rng.uniform_int(3)
        for _ in range(pre):
            eps = eps + np.array([rng.uniform(-0.03, 0.03), rng.uniform(-0.03, 0.03), rng.uniform(-0.05, 0.05)])
            st = O.update_material(mat, st, eps)[2]
        probe = eps + np.array([rng.uniform(-0.03, 0.03), rng.uniform(-0.03, 0.03), rng.uniform(-0.05, 0.05)])
        s4, _, st4 = O.update4(mat, st, np.array([probe[0], probe[1], 0.0, 0.5 * probe[2]]))
        dlam = st4[4] - st[4]
        if 0.0 < dlam < 60e-6:
            continue
        if dlam == 0.0 and mat[0] == "j2":
            x = np.array([probe[0], probe[1], 0.0, 0.5 * probe[2]]) - st[:4]
            lam = 0.3 / (1.3 * 0.4)
            t = lam * x[:3].sum() * np.array([1, 1, 1, 0.0]) + 2 * mu * x
            q_tr = vonmises4(t)
            if q_tr > 0.01 + 0.016 * st[4] - 60e-6 * 3 * mu:
                continue
        s, C, st_new, _ = O.update_material(mat, st, probe)
        h = 1e-6
        fd = np.zeros((3, 3))
        for j in range(3):
            ep, em = probe.copy(), probe.copy()
            ep[j] += h
            em[j] -= h
            fd[:, j] = (O.update_material(mat, st, ep)[0] - O.update_material(mat, st, em)[0]) / (2 * h)
        assert np.abs(C - fd).max() / np.abs(C).max() < 1e-6, (name, tested)
        deps = st_new[:4] - st[:4]
        assert abs(deps[:3].sum()) < 1e-10
        assert st_new[4] >= st[4]
        sig4 = np.array([s[0], s[1], st_new[5], s[2]])
        assert sig4[0] * deps[0] + sig4[1] * deps[1] + sig4[2] * deps[2] + 2 * sig4[3] * deps[3] >= -1e-12
        tested += 1
    assert tested == 120


DESK = [J2, ("elastic", 10.0, 0.3)]  # desk_materials (test_rve.cpp:9-17)


def test_homogeneous_rve_zero_fluctuation_exact_response():
    """test_rve.cpp:44-62 (linear BC)"""
    mesh = O.Mesh(geometry=1, subdivisions=4)
    E = np.array([0.01, -0.004, 0.006])
    r = mesh.hf_trajectory([("elastic", 2.0, 0.25)], E[None, :])
    assert r["iterations"][0] <= 1
    assert r["u_fluct_inf"][0] < 1e-10
    C = elastic_C(2.0, 0.25)
    assert np.linalg.norm(r["sigma"][0] - C @ E) < 1e-8 * np.linalg.norm(C @ E)
    assert np.abs(r["C"][0] - C).max() < 1e-8 * np.abs(C).max()


def test_elastic_load_one_iteration_repeat_zero():
    """test_rve.cpp:82-100 — an elastic load converges in exactly one Newton
    iteration; re-solving the converged state at tol 1e-10 takes zero."""
    mesh = O.Mesh(0, 6)
    E = np.array([0.001, 0.0, 0.0])
    r = mesh.hf_trajectory(DESK, np.stack([E, E]), tol=1e-10)
    assert list(r["iterations"]) == [1, 0]


def test_mesh_counts_and_area():
    """mesh.hpp:218-352: default_cell(33) — the BASELINE config-0 RVE
    (~2,000 Tri6 elements); area within 2% of 1 - pi 0.15^2 (test_mesh.cpp)."""
    m = O.Mesh(0, 33)
    assert (m.n_elements, m.n_nodes) == (2025, 4219)
    assert abs(m.area - (1 - np.pi * 0.15 ** 2)) < 0.02
    # every IP has a positive Jacobian and B reproduces an affine field (patch test, test_mesh.cpp:67-87)
    E = np.array([0.01, -0.02, 0.03])
    for ip in range(0, 3 * m.n_elements, 97):
        B, w, e = m.ip(ip)
        assert w > 0
        xy = m.xy[m.conn[e]]
        u = np.zeros(12)
        u[0::2] = E[0] * xy[:, 0] + 0.5 * E[2] * xy[:, 1]
        u[1::2] = 0.5 * E[2] * xy[:, 0] + E[1] * xy[:, 1]
        assert np.abs(B @ u - E).max() < 1e-10


@pytest.mark.parametrize("elastic", [True, False])
def test_hf_condensed_tangent_matches_fd(elastic):
    """test_rve.cpp:132-161 (heterogeneous elastic) and :163-195 (plastic):
    C_hom vs central FD of Σ(E), rel < 1e-5; symmetric to 1e-8."""
    mesh = O.Mesh(0, 6)
    mats = [("elastic", 1.0, 0.3), ("elastic", 10.0, 0.3)] if elastic else DESK
    if elastic:
        pre, E = [], np.array([0.012, -0.003, 0.008])
    else:
        pre, E = [np.array([0.02, 0.005, -0.015])], np.array([0.025, 0.005, -0.018])
    path = np.array(pre + [E])
    r = mesh.hf_trajectory(mats, path, tol=1e-12)
    C = r["C"][-1]
    h = 1e-6
    fd = np.zeros((3, 3))
    for j in range(3):
        ep, em = E.copy(), E.copy()
        ep[j] += h
        em[j] -= h
        sp = mesh.hf_trajectory(mats, np.array(pre + [ep]), tol=1e-12)["sigma"][-1]
        sm = mesh.hf_trajectory(mats, np.array(pre + [em]), tol=1e-12)["sigma"][-1]
        fd[:, j] = (sp - sm) / (2 * h)
    assert np.abs(C - fd).max() < 1e-5 * np.abs(C).max()
    if elastic:
        assert np.abs(C - C.T).max() < 1e-8 * np.abs(C).max()
