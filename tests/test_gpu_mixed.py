"""Mixed control on the hyper-ROM engine (fe2_hrom_mixed_step; rve.hpp:496-571
mixed_control_step): the reference's own test case (test_rve.cpp:310-322,
uniaxial tension drives the transverse stresses to zero, lateral contraction)
for every point, and the replay property — the accepted states are exactly
those of a plain increment run along the converged macro strains."""
import numpy as np
import pytest

import paper_2306_02687_b200 as F

pytestmark = pytest.mark.gpu


def _engine(P, n=12, K=200):
    eng = F.HyperRomEngine.from_model(F.HyperRomModel(33, n, K, 0))
    eng.alloc_points(P)
    return eng


def test_uniaxial_tension_drives_transverse_stresses_to_zero():
    P = 16
    eng = _engine(P)
    rng = np.random.default_rng(0)
    scale = rng.uniform(0.5, 1.5, P)  # different load levels per point
    E = np.zeros((P, 3))
    path = []
    for k in range(1, 6):
        Ep = np.zeros((P, 3))
        Ep[:, 0] = 0.02 * k / 5.0 * scale
        o = eng.mixed_step([True, False, False], Ep, np.zeros((P, 3)), E)
        assert (o["status"] == 0).all()
        assert np.abs(o["sigma"][:, 1:]).max() < 1e-10
        assert (o["outer_iters"] >= 1).all()
        E = o["E"]
        path.append((E.copy(), o["sigma"].copy(), o["C"].copy()))
    assert (path[-1][1][:, 0] > 0).all()
    assert (E[:, 1] < 0).all()  # lateral contraction
    # replay: the accepted states are those of plain increments along the converged strains
    ref = _engine(P)
    for Ek, sk, Ck in path:
        r = ref.solve_increment(Ek)
        np.testing.assert_array_equal(r["sigma"], sk)
        np.testing.assert_array_equal(r["C"], Ck)


def test_fully_prescribed_is_a_plain_increment():
    P = 8
    eng, ref = _engine(P), _engine(P)
    Ep = F.make_paths(0, 0, P, 1)[:, 0]
    o = eng.mixed_step([True, True, True], Ep, np.zeros((P, 3)), np.zeros((P, 3)))
    r = ref.solve_increment(Ep)
    assert (o["outer_iters"] == 0).all() and (o["status"] == 0).all()
    np.testing.assert_array_equal(o["E"], Ep)
    np.testing.assert_array_equal(o["sigma"], r["sigma"])


def test_stress_target_and_mixed_masks():
    """Per-point masks: pure stress control hits an arbitrary target; the
    unknown components move only where they are unknown."""
    P = 4
    eng = _engine(P)
    ctl = np.array([[False, False, False], [True, False, True], [False, True, False], [True, True, False]])
    tgt = np.array([[0.004, -0.002, 0.001], [0.0, 0.003, 0.0], [0.002, 0.0, -0.001], [0.0, 0.0, 0.0015]])
    Ep = np.array([[0.0, 0.0, 0.0], [0.004, 0.0, 0.002], [0.0, -0.003, 0.0], [0.003, 0.001, 0.0]])
    o = eng.mixed_step(ctl, Ep, tgt, np.zeros((P, 3)))
    assert (o["status"] == 0).all()
    for p in range(P):
        u = ~ctl[p]
        assert np.abs(o["sigma"][p][u] - tgt[p][u]).max() < 1e-10 * (np.linalg.norm(tgt[p]) + 1e-3)
        np.testing.assert_array_equal(o["E"][p][ctl[p]], Ep[p][ctl[p]])


def test_mixed_control_on_the_cta_kernel_and_power_law():
    """n = 64 (k_increment_big) with a power-law matrix: uniaxial stress, the replay property."""
    P = 8
    m = F.HyperRomModel(33, 64, 1000, 0)
    m.materials = [F.PowerLawParams(1.0, 0.3, 0.01, 0.1), F.ElasticParams(10.0, 0.3)]
    eng = F.HyperRomEngine.from_model(m)
    eng.alloc_points(P)
    E = np.zeros((P, 3))
    steps = []
    for k in range(1, 4):
        Ep = np.zeros((P, 3))
        Ep[:, 0] = 0.015 * k
        o = eng.mixed_step([True, False, False], Ep, np.zeros((P, 3)), E)
        assert (o["status"] == 0).all() and np.abs(o["sigma"][:, 1:]).max() < 1e-10
        E = o["E"]
        steps.append((E.copy(), o["sigma"].copy()))
    ref = F.HyperRomEngine.from_model(m)
    ref.alloc_points(P)
    for Ek, sk in steps:
        np.testing.assert_array_equal(ref.solve_increment(Ek)["sigma"], sk)


def test_mixed_control_failure_status():
    """max_iter = 0 cannot move the unknown components: status 1 + solver for the
    points with an unmet target, 0 for the fully prescribed one."""
    P = 3
    eng = _engine(P)
    ctl = np.array([[True, False, False], [True, True, True], [False, False, False]])
    Ep = np.array([[0.01, 0.0, 0.0], [0.002, 0.001, 0.0], [0.0, 0.0, 0.0]])
    tgt = np.array([[0.0, 0.0, 0.0], [0.0, 0.0, 0.0], [0.003, 0.0, 0.0]])
    o = eng.mixed_step(ctl, Ep, tgt, np.zeros((P, 3)), max_iter=0)
    assert o["status"][0] == 1 + 4 and o["status"][2] == 1 + 4 and o["status"][1] == 0
