"""Power-law and creep material points on the device (materials.hpp:216-292;
SURVEY §8(f) rank 4): the batched update and the HF RVE solver against the
oracle's restatement."""
import numpy as np
import pytest

import pyoracle as O
import paper_2306_02687_b200 as F
from paper_2306_02687_b200 import pod as P

pytestmark = pytest.mark.gpu


def _states(rng, N, eq_max=0.02):
    state = np.zeros((N, 6))
    state[:, :4] = rng.uniform(-0.01, 0.01, size=(N, 4))
    state[:, 2] = -(state[:, 0] + state[:, 1])
    state[:, 4] = rng.uniform(0.0, eq_max, size=N)
    return state


@pytest.mark.parametrize("mat", [F.PowerLawParams(1.01, 0.29, 0.0072, 0.08), F.PowerLawParams(1.0, 0.3, 0.01, 0.3),
                                 F.CreepParams(dt=0.7), F.CreepParams(1.0, 0.3, 5.0, 1.2, 0.0, 0.1)])
def test_material_batch_matches_oracle(mat):
    rng = np.random.default_rng(11)
    N = 4096
    eps = rng.uniform(-0.03, 0.03, size=(N, 3))
    state = _states(rng, N)
    sig, C, so, pl = F.update_material_batch(mat, eps, state)
    n_pl = 0
    for i in range(0, N, 5):
        s_o, C_o, so_o, pl_o = O.update_material(mat, state[i], eps[i])
        assert pl[i] == pl_o
        n_pl += pl_o
        np.testing.assert_allclose(sig[i], s_o, rtol=1e-11, atol=1e-15)
        np.testing.assert_allclose(C[i], C_o, rtol=1e-9, atol=1e-12 * np.abs(C_o).max())
        np.testing.assert_allclose(so[i], so_o, rtol=1e-11, atol=1e-15)
    assert n_pl > 50


def test_creep_without_dt_is_material_error():
    with pytest.raises(F.Fe2Error) as e:
        F.update_material_batch(F.CreepParams(dt=0.0), np.array([[0.01, 0.0, 0.0]]))
    assert e.value.code == 4  # 1 + ErrorCode::material


def test_engine_material_rules():
    """The small-strain engine takes one inelastic (J2 / power law / creep) material per
    model (the iterative ones through general_return, tests/test_gpu_general_materials.py);
    two distinct inelastic materials, or an iterative one on the finite-strain handle,
    are configuration errors."""
    m = F.HyperRomModel(8, 4, 20, 0)
    F.HyperRomEngine(m.G, m.w, m.mat, [F.PowerLawParams(), F.ElasticParams(10.0, 0.3)], m.volume).close()
    mid = m.mat.copy()
    mid[mid == 1] = 2  # the inclusions get a second inelastic material
    with pytest.raises(F.Fe2Error) as e:
        F.HyperRomEngine(m.G, m.w, mid, [F.PowerLawParams(), F.ElasticParams(10.0, 0.3), F.CreepParams()], m.volume)
    assert e.value.code == 1
    with pytest.raises(F.Fe2Error) as e:
        F.HyperRomEngine(m.G4, m.w, m.mat, [F.PowerLawParams(), F.ElasticParams(10.0, 0.3)], m.volume)
    assert e.value.code == 1


@pytest.mark.parametrize("matrix,tol", [(F.PowerLawParams(1.0, 0.3, 0.01, 0.1), 1e-8), (F.CreepParams(1.0, 0.3, 5.0, 1.2, -0.3, 0.5), 1e-8)])
def test_hf_trajectory_matches_oracle(matrix, tol):
    """Full-field RVE with a power-law / creep matrix: identical Newton
    iteration counts (bisections scale the creep dt), Σ / C within 1e-9."""
    mats = [matrix, F.ElasticParams(10.0, 0.3)]
    path = np.array([[0.004, -0.001, 0.002], [0.010, -0.003, 0.006], [0.02, -0.006, 0.012], [0.012, -0.004, 0.006]])
    opts = F.NewtonOptions(tol, 30, 6)
    g = P.HfRve(8, materials=mats).trajectory(path, opts)
    o = O.Mesh(0, 8).hf_trajectory(mats, path, tol=tol, max_iter=30, max_bisections=6, snapshots=True)
    np.testing.assert_array_equal(g["iterations"], o["iterations"])
    assert np.abs(g["sigma"] - o["sigma"]).max() < 1e-9 * np.abs(o["sigma"]).max()
    assert np.abs(g["C"] - o["C"]).max() < 1e-9 * np.abs(o["C"]).max()
    assert np.abs(g["snapshots"] - o["snapshots"]).max() < 1e-8 * np.abs(o["snapshots"]).max()
