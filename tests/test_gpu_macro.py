"""The device macro driver (fe2_macro_run: host C++ macro Newton + one engine
increment per macro iteration, snapshot/restore for the nested micro
commit) against the oracle driver (numpy macro Newton + replayed oracle
hyper-ROM) on the desk beam: identical step sequence and macro iteration
counts, reactions within 1e-8 relative, same residual displacement. The
micro solves see macro strains that differ from the oracle's by rounding
(1e-13 relative, accumulated through the macro Newton), so a micro point
sitting on a convergence-test knife edge may take one more or fewer Newton
iteration: cumulative micro counts agree to 1e-3 (the hot-path tests pin
exact counts on identical inputs)."""
import numpy as np
import pytest

import macro_oracle as MO
import paper_2306_02687_b200 as F
import pyoracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("u_max,n_load", [(0.02, 5), (0.3, 10)])
def test_device_macro_driver_matches_oracle(u_max, n_load):
    m = F.HyperRomModel(33, 12, 200, 0)
    eng = F.HyperRomEngine.from_model(m)
    cfg = F.MacroConfig(u_max=u_max, n_load=n_load)
    g = F.solve_program(cfg, eng)
    beam = MO.build_beam(cfg.length, cfg.height, cfg.nx, cfg.ny)
    orc = O.Hrom(m.G, m.w, m.mat, m.materials, m.volume)
    rows, ures = MO.solve_program(beam, MO.ReplayEngine(orc, len(beam["w"]), threads=16), u_max=u_max,
                                  n_load=n_load, max_unload=cfg.max_unload, tol=cfg.tol, max_iter=cfg.max_iter)
    assert len(g["U"]) == len(rows)
    np.testing.assert_allclose(g["U"], rows[:, 0], rtol=0, atol=1e-15)
    np.testing.assert_array_equal(g["macro_iters"], rows[:, 2].astype(int))
    np.testing.assert_allclose(g["micro_iters"], rows[:, 3], rtol=1e-3, atol=0)
    scale = np.abs(rows[:, 1]).max()
    assert np.abs(g["R"] - rows[:, 1]).max() <= 1e-8 * scale
    if u_max > 0.1:
        assert g["U_residual"] > 0.0
    assert abs(g["U_residual"] - ures) <= 1e-8 * u_max


def test_device_finite_strain_macro_driver_matches_oracle():
    """Total-Lagrangian FE² beam on the finite-strain engine (config-2
    kinematics) against the oracle driver on the finite-strain oracle."""
    m = F.HyperRomModel(33, 12, 200, 0)
    eng = F.HyperRomEngine.from_model(m, finite_strain=True)
    cfg = F.MacroConfig(u_max=0.3, n_load=10)
    g = F.solve_program(cfg, eng)
    beam = MO.build_beam(cfg.length, cfg.height, cfg.nx, cfg.ny)
    orc = O.HromFs(m.G4, m.w, m.mat, m.materials, m.volume)
    rows, ures = MO.solve_program(beam, MO.ReplayEngine(orc, len(beam["w"]), threads=16), u_max=cfg.u_max,
                                  n_load=cfg.n_load, max_unload=cfg.max_unload, tol=cfg.tol, max_iter=cfg.max_iter)
    assert len(g["U"]) == len(rows)
    np.testing.assert_array_equal(g["macro_iters"], rows[:, 2].astype(int))
    np.testing.assert_allclose(g["micro_iters"], rows[:, 3], rtol=1e-3, atol=0)
    assert np.abs(g["R"] - rows[:, 1]).max() <= 1e-8 * np.abs(rows[:, 1]).max()
    assert g["U_residual"] > 0.0 and abs(g["U_residual"] - ures) <= 1e-8 * cfg.u_max


@pytest.mark.parametrize("u_max,n_load,n,K", [(0.02, 3, 12, 200), (0.3, 10, 12, 200), (0.3, 6, 40, 300),
                                             (0.3, 4, 64, 500), (0.3, 3, 128, 600)])
def test_device_monolithic_driver_matches_oracle(u_max, n_load, n, K):
    """Monolithic scheme (fe2_hrom_mono_*): the device macro driver against
    the oracle's monolithic driver — identical steps and macro iteration
    counts, micro iterations = P per macro iteration, R within 1e-8. n = 12
    runs the warp-per-point kernel, n = 40 / 64 / 128 the CTA-per-point one
    (4- and 8-warp CTAs)."""
    m = F.HyperRomModel(33, n, K, 0)
    eng = F.HyperRomEngine.from_model(m)
    cfg = F.MacroConfig(u_max=u_max, n_load=n_load, scheme="monolithic")
    g = F.solve_program(cfg, eng)
    beam = MO.build_beam(cfg.length, cfg.height, cfg.nx, cfg.ny)
    orc = O.Hrom(m.G, m.w, m.mat, m.materials, m.volume)
    rows, ures = MO.solve_program(beam, MO.MonoEngine(orc, len(beam["w"]), m.volume), u_max=u_max, n_load=n_load,
                                  max_unload=cfg.max_unload, tol=cfg.tol, max_iter=cfg.max_iter,
                                  micro_tol=cfg.micro.tol)
    assert len(g["U"]) == len(rows)
    np.testing.assert_allclose(g["U"], rows[:, 0], rtol=0, atol=1e-15)
    np.testing.assert_array_equal(g["macro_iters"], rows[:, 2].astype(int))
    np.testing.assert_array_equal(g["micro_iters"], rows[:, 3])
    assert np.abs(g["R"] - rows[:, 1]).max() <= 1e-8 * np.abs(rows[:, 1]).max()
    assert abs(g["U_residual"] - ures) <= 1e-8 * u_max


def test_device_monolithic_reaches_the_nested_fixed_point():
    """same R(U) curve and residual displacement as the nested
    scheme (within the tolerances), with far fewer micro iterations."""
    m = F.HyperRomModel(33, 12, 200, 0)
    nested = F.solve_program(F.MacroConfig(u_max=0.3, n_load=10), F.HyperRomEngine.from_model(m))
    mono = F.solve_program(F.MacroConfig(u_max=0.3, n_load=10, scheme="monolithic"), F.HyperRomEngine.from_model(m))
    assert len(mono["U"]) == len(nested["U"])
    assert np.abs(mono["R"] - nested["R"]).max() < 1e-5 * np.abs(nested["R"]).max()
    assert abs(mono["U_residual"] - nested["U_residual"]) < 1e-4 * 0.3
