"""Macro FE driver of the two-scale beam (SPEC.md:455-518,
nested variant): the product's beam mesh / Gauss-point operators against the
oracle restatement, the patch test, and the oracle driver's SPEC properties
(elastic reversibility U_res = 0, plastic U_res > 0, monotone R on loading).
The device driver is compared with the oracle driver in test_gpu_macro.py."""
import numpy as np
import pytest

import macro_oracle as MO
import paper_2306_02687_b200 as F
import pyoracle as O


@pytest.mark.parametrize("L,H,nx,ny", [(4.0, 1.0, 8, 2), (2.0, 0.5, 3, 1)])
def test_beam_gauss_operators_match_oracle(L, H, nx, ny):
    cfg = F.MacroConfig(length=L, height=H, nx=nx, ny=ny)
    B, w, e = F.macro_gauss(cfg)
    beam = MO.build_beam(L, H, nx, ny)
    assert len(w) == 3 * 2 * nx * ny
    np.testing.assert_allclose(B, beam["B"], rtol=0, atol=1e-12 * np.abs(B).max())
    np.testing.assert_allclose(w, beam["w"], rtol=1e-14)
    np.testing.assert_array_equal(e, beam["elem"])
    assert abs(w.sum() - L * H) < 1e-12 * L * H


def test_patch_test_uniform_strain():
    """u = E·x reproduces E at every macro Gauss point (test_mesh.cpp:67-87 pattern)."""
    beam = MO.build_beam(4.0, 1.0, 8, 2)
    E = np.array([0.01, -0.004, 0.006])  # (E11, E22, 2E12)
    xy = beam["xy"]
    u = np.zeros(2 * len(xy))
    u[0::2] = E[0] * xy[:, 0] + 0.5 * E[2] * xy[:, 1]
    u[1::2] = 0.5 * E[2] * xy[:, 0] + E[1] * xy[:, 1]
    B, _, elem = F.macro_gauss(F.MacroConfig())
    tri = beam["tri"]
    for g in range(len(elem)):
        dofs = [2 * tri[elem[g]][d // 2] + d % 2 for d in range(12)]
        np.testing.assert_allclose(B[g] @ u[dofs], E, atol=1e-14)


@pytest.fixture(scope="module")
def desk_hrom():
    md = O.Model(subdivisions=33, n=12, K=200, seed=0)
    desk = [("j2", 1.0, 0.3, 0.01, 0.016), ("elastic", 10.0, 0.3)]
    return O.Hrom(md.G, md.w, md.mat, desk, md.volume)


def test_oracle_driver_elastic_reversible(desk_hrom):
    beam = MO.build_beam(4.0, 1.0, 8, 2)
    rows, ures = MO.solve_program(beam, MO.ReplayEngine(desk_hrom, len(beam["w"])), u_max=0.02, n_load=5)
    load = rows[:5]
    np.testing.assert_allclose(load[:, 1] / load[:, 0], load[0, 1] / load[0, 0], rtol=1e-6)  # linear R(U)
    assert abs(ures) < 1e-6 * 0.02


def test_oracle_driver_plastic_residual_displacement(desk_hrom):
    beam = MO.build_beam(4.0, 1.0, 8, 2)
    rows, ures = MO.solve_program(beam, MO.ReplayEngine(desk_hrom, len(beam["w"])), u_max=0.3, n_load=6)
    load = rows[:6]
    assert (np.diff(load[:, 1]) > 0).all()  # hardening: R non-decreasing while loading
    secant = load[:, 1] / load[:, 0]
    assert secant[-1] < 0.98 * secant[0]  # yielding softens the response
    assert 0.0 < ures < 0.3
    # the step predictor (last accepted tangent) is exact for elastic steps;
    # plastic loading steps still iterate
    assert (rows[:, 2] >= 0).all() and load[:, 2].max() >= 1


def test_oracle_finite_strain_driver_small_load_limit():
    """Total-Lagrangian FE² with the finite-strain oracle: for a small tip
    displacement the reaction equals the small-strain driver's to O(U)."""
    md = O.Model(subdivisions=33, n=12, K=200, seed=0)
    desk = [("j2", 1.0, 0.3, 0.01, 0.016), ("elastic", 10.0, 0.3)]
    G4 = O.model_g4(33, 12, 200, 0)
    beam = MO.build_beam(4.0, 1.0, 8, 2)
    ss = O.Hrom(md.G, md.w, md.mat, desk, md.volume)
    fs = O.HromFs(G4, md.w, md.mat, desk, md.volume)
    r_ss, _ = MO.solve_program(beam, MO.ReplayEngine(ss, len(beam["w"])), u_max=1e-3, n_load=2, max_unload=0)
    r_fs, _ = MO.solve_program(beam, MO.ReplayEngine(fs, len(beam["w"])), u_max=1e-3, n_load=2, max_unload=0)
    np.testing.assert_allclose(r_fs[:, 1], r_ss[:, 1], rtol=5e-3)


def test_oracle_monolithic_reaches_the_nested_fixed_point(desk_hrom):
    """the monolithic scheme converges to the nested scheme's
    fixed point (same R(U) curve and U_res within the tolerances); every
    accepted step has all micro residuals below micro tol."""
    beam = MO.build_beam(4.0, 1.0, 8, 2)
    P = len(beam["w"])
    kw = dict(u_max=0.3, n_load=5, max_unload=30)
    rn, un = MO.solve_program(beam, MO.ReplayEngine(desk_hrom, P), **kw)
    rm, um = MO.solve_program(beam, MO.MonoEngine(desk_hrom, P, desk_hrom_volume()), **kw)
    assert len(rn) == len(rm)
    np.testing.assert_allclose(rm[:, 0], rn[:, 0], rtol=0, atol=1e-12)
    assert np.abs(rm[:, 1] - rn[:, 1]).max() < 1e-5 * np.abs(rn[:, 1]).max()
    assert abs(um - un) < 1e-4 * 0.3
    assert um > 0


def test_oracle_monolithic_elastic_equals_nested(desk_hrom):
    beam = MO.build_beam(4.0, 1.0, 8, 2)
    P = len(beam["w"])
    rn, _ = MO.solve_program(beam, MO.ReplayEngine(desk_hrom, P), u_max=0.02, n_load=3, max_unload=0)
    rm, _ = MO.solve_program(beam, MO.MonoEngine(desk_hrom, P, desk_hrom_volume()), u_max=0.02, n_load=3,
                             max_unload=0)
    np.testing.assert_allclose(rm[:, 1], rn[:, 1], rtol=1e-8)


def desk_hrom_volume():
    return O.Model(subdivisions=33, n=12, K=200, seed=0).volume
