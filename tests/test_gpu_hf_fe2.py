"""Full-field HF FE² (fe2_macro_run_hf; SPEC.md:474-477 HF_nested) on the
device HF engine: the per-point increments equal run_trajectory, and the
hyper-ROM FE² agrees with it — exactly in the elastic range on the elastic
modes ("elastic load, all methods → identical R"), and within
the SPEC's method-agreement tolerance on POD bases in the plastic range."""
import numpy as np
import pytest

import paper_2306_02687_b200 as F
from paper_2306_02687_b200 import pod as P

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rve8():
    return P.HfRve(8)


def test_hf_engine_increments_equal_trajectories(rve8):
    rng = np.random.default_rng(3)
    paths = np.cumsum(rng.uniform(-0.004, 0.006, size=(3, 5, 3)), axis=1)
    ref = [rve8.trajectory(paths[p], snapshots=False) for p in range(3)]
    rve8.alloc_points(3)
    for k in range(5):
        out = rve8.solve_increment(paths[:, k])
        assert (out["status"] == 0).all()
        for p in range(3):
            np.testing.assert_array_equal(out["sigma"][p], ref[p]["sigma"][k])
            np.testing.assert_array_equal(out["C"][p], ref[p]["C"][k])
            assert out["iters"][p] == ref[p]["iterations"][k]


def test_hf_engine_snapshot_restore(rve8):
    rve8.alloc_points(2)
    E1 = np.array([[0.01, 0.0, 0.004], [0.0, -0.01, 0.006]])
    a = rve8.solve_increment(E1)
    rve8.snapshot()
    b = rve8.solve_increment(2 * E1)
    rve8.restore()
    c = rve8.solve_increment(2 * E1)
    np.testing.assert_array_equal(b["sigma"], c["sigma"])
    assert not np.array_equal(a["sigma"], b["sigma"])


def test_elastic_fe2_hf_equals_hyper_rom_on_elastic_modes(rve8):
    cfg = F.MacroConfig(u_max=0.02, n_load=3, max_unload=0)
    hf = F.solve_program(cfg, rve8)
    md = F.HyperRomModel(8, K=0, basis=rve8.elastic_modes())
    g = F.solve_program(cfg, F.HyperRomEngine.from_model(md))
    assert len(g["U"]) == len(hf["U"]) == 3
    np.testing.assert_allclose(g["R"], hf["R"], rtol=1e-8)


def test_plastic_fe2_hyper_rom_pod_agrees_with_hf(rve8):
    """Method agreement: hyper-ROM FE² on a 24-mode POD basis
    (30 monotonic HF training trajectories, full rule) reproduces the HF FE²
    load curve within 1% and the residual displacement within 1% of Ū."""
    cfg = F.MacroConfig(u_max=0.3, n_load=10)
    hf = F.solve_program(cfg, rve8)
    rng = np.random.default_rng(1)
    ends = rng.standard_normal((30, 3))
    ends *= 0.03 / np.linalg.norm(ends, axis=1, keepdims=True)
    X, _ = P.collect_snapshots(rve8, ends, 10)
    V, _, _ = P.pod_basis(X, 24, rve8.elastic_modes())
    g = F.solve_program(cfg, F.HyperRomEngine.from_model(F.HyperRomModel(8, K=0, basis=V)))
    assert F.fe2.curve_error(g, hf) < 0.01
    assert abs(g["U_residual"] - hf["U_residual"]) < 0.01 * cfg.u_max
    assert hf["U_residual"] > 0
