"""The oracle's power-law and strain-hardening-creep material points
(materials.hpp:51-76, :216-292) against the reference's own known-answer
tests (test_materials.cpp:120-271): zero-increment identity, the N -> 0
perfect-plasticity limit, monotone concave hardening, creep at zero stress,
Norton (m = 0) independence of the creep history, the analytic
strain-hardening solution under constant stress, and consistent tangents
against central finite differences with the flow invariants."""
import numpy as np
import pytest

import pyoracle as O

PL = ("powerlaw", 1.01, 0.29, 0.0072, 0.08)


def creep(dt, E=1.0, nu=0.14, A=22.09, n=1.06, m=-0.56):
    return ("creep", E, nu, A, n, m, dt)


def vonmises4(s):
    p = s[:3].sum() / 3.0
    d = np.array([s[0] - p, s[1] - p, s[2] - p, s[3]])
    return np.sqrt(1.5 * (d[0] ** 2 + d[1] ** 2 + d[2] ** 2 + 2 * d[3] ** 2))


def sigma4(s3, st):
    return np.array([s3[0], s3[1], st[5], s3[2]])


def test_power_law_zero_increment_identity():
    s0 = np.array([0.001, -0.0005, -0.0005, 0.0002, 0.0015, 0.0])
    e = np.array([0.0008, -0.0002, 0.0001])
    s, _, st, _ = O.update_material(PL, s0, e)
    s2, _, st2, _ = O.update_material(PL, st, e)
    assert abs(st2[4] - st[4]) <= 1e-14
    assert np.linalg.norm(s2 - s) < 1e-12


def test_power_law_small_N_is_perfect_plasticity():
    mat = ("powerlaw", 1.0, 0.3, 0.01, 1e-9)
    st = np.zeros(6)
    for k in range(1, 11):
        s, _, st, _ = O.update_material(mat, st, np.array([0.06 * k / 10, 0.0, 0.01 * k / 10]))
        if st[4] > 0:
            assert abs(vonmises4(sigma4(s, st)) - 0.01) < 1e-6 * 0.01
    assert st[4] > 0


def test_power_law_monotone_concave_hardening():
    mat = ("powerlaw", 1.01, 0.29, 0.72 * 0.01, 0.08)
    st = np.zeros(6)
    eqs, qs = [], []
    for k in range(1, 31):
        s, _, st, _ = O.update_material(mat, st, np.array([0.1 * k / 30, 0.0, 0.0]))
        if st[4] > 1e-12:
            eqs.append(st[4])
            qs.append(vonmises4(sigma4(s, st)))
    assert len(eqs) >= 10
    assert all(b > a for a, b in zip(qs, qs[1:]))
    for i in range(2, len(qs)):
        prev = (qs[i - 1] - qs[i - 2]) / (eqs[i - 1] - eqs[i - 2])
        cur = (qs[i] - qs[i - 1]) / (eqs[i] - eqs[i - 1])
        assert cur < prev * (1 + 1e-9)


def test_creep_zero_stress_unchanged():
    s0 = np.array([0.002, -0.001, -0.001, 0.0, 0.002, 0.0])
    s, _, st = O.update4(creep(0.5), s0, s0[:4])
    assert st[4] == s0[4]
    assert np.linalg.norm(s) < 1e-12


def test_creep_norton_rate_independent_of_history():
    mat = creep(0.1, 1.0, 0.3, 5.0, 1.2, 0.0)
    eps = np.array([0.01, -0.002, 0.0, 0.003])
    _, _, r1 = O.update4(mat, np.zeros(6), eps)
    aged = np.zeros(6)
    aged[4] = 0.5
    _, _, r2 = O.update4(mat, aged, eps)
    assert r1[4] - 0.0 == pytest.approx(r2[4] - 0.5, rel=1e-10)


def test_creep_constant_stress_matches_analytic_strain_hardening():
    A, n, m, E, nu = 22.09, 1.06, -0.56, 1.0, 0.14
    sig, T, steps = 0.01 * A, 100.0, 100
    target = np.array([sig, 0.0, 0.0, 0.0])
    st = np.zeros(6)
    eps = np.array([sig / E, -nu * sig / E, -nu * sig / E, 0.0])
    mat = creep(T / steps)
    for _ in range(steps):
        for _ in range(60):  # stress-controlled strain (mixed control, full 4-component Newton)
            s4, D, _ = O.update4(mat, st, eps)
            r = target - s4
            if np.abs(r).max() <= 1e-13 * sig:
                break
            eps = eps + np.linalg.solve(D, r)
        _, _, st_new = O.update4(mat, st, eps)
        assert st_new[4] >= st[4]
        st = st_new
    exact = (sig / A) ** n * T ** (m + 1) / (m + 1)
    assert abs(st[4] - exact) / exact < 0.01


@pytest.mark.parametrize("name", ["powerlaw", "creep"])
def test_consistent_tangent_matches_central_fd(name):
    """test_materials.cpp:210-271 for the power law and creep: 120 states
    from Rng(42), rel < 1e-6, deviatoric flow, eq monotone, dissipation >= 0."""
    rng = O.Rng(42)
    tested = guard = 0
    E, nu = (1.01, 0.29) if name == "powerlaw" else (1.0, 0.14)
    lam, mu = E * nu / ((1 + nu) * (1 - 2 * nu)), E / (2 * (1 + nu))
    while tested < 120 and guard < 5000:
        guard += 1
        st = np.zeros(6)
        eps = np.zeros(3)
        dt = 0.5 + rng.uniform()
        mat = PL if name == "powerlaw" else creep(dt)
        pre = rng.uniform_int(3)
        ok = True
        for _ in range(pre):
            eps = eps + np.array([rng.uniform(-0.03, 0.03), rng.uniform(-0.03, 0.03), rng.uniform(-0.05, 0.05)])
            if ok:
                try:
                    st = O.update_material(mat, st, eps)[2]
                except O.OracleError:
                    ok = False
        probe = eps + np.array([rng.uniform(-0.03, 0.03), rng.uniform(-0.03, 0.03), rng.uniform(-0.05, 0.05)])
        if not ok:
            continue
        e4 = np.array([probe[0], probe[1], 0.0, 0.5 * probe[2]])
        _, _, st4 = O.update4(mat, st, e4)
        dlam = st4[4] - st[4]
        if 0.0 < dlam < 60e-6:
            continue
        if dlam == 0.0 and name == "powerlaw":
            x = e4 - st[:4]
            t = lam * x[:3].sum() * np.array([1, 1, 1, 0.0]) + 2 * mu * x
            sy = 0.0072 * (1 + 1.01 * st[4] / 0.0072) ** 0.08
            if vonmises4(t) > sy - 60e-6 * 3 * mu:
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
        sig4 = sigma4(s, st_new)
        assert sig4[0] * deps[0] + sig4[1] * deps[1] + sig4[2] * deps[2] + 2 * sig4[3] * deps[3] >= -1e-12
        tested += 1
    assert tested == 120


def test_invalid_parameters_rejected():
    for bad in [("powerlaw", 1.0, 0.3, 0.01, 1.5), ("powerlaw", 1.0, 0.3, -1.0, 0.1), creep(1.0, m=-1.5),
                creep(1.0, A=0.0)]:
        with pytest.raises(O.OracleError):
            O.update_material(bad, None, np.array([0.01, 0.0, 0.0]))
    with pytest.raises(O.OracleError):
        O.update_material(creep(0.0), None, np.array([0.01, 0.0, 0.0]))
