"""POD basis from HF snapshots on the device: the
device HF solver (fe2_hf_trajectory) against the oracle's micro_newton /
homogenize / run_trajectory restatement, elastic modes, the device POD
against the numpy POD oracle, and the ROM -> HF convergence of hyper-ROM
models built on the physical basis."""
import numpy as np
import pytest

import pod_oracle as PO
import pyoracle as O
import paper_2306_02687_b200 as F
from paper_2306_02687_b200 import pod as P

pytestmark = pytest.mark.gpu

DESK = [("j2", 1.0, 0.3, 0.01, 0.016), ("elastic", 10.0, 0.3)]
PATH = np.array([[0.004, -0.001, 0.002], [0.008, -0.002, 0.004], [0.016, -0.004, 0.009], [0.010, -0.003, 0.005],
                 [0.0, 0.0, 0.0], [-0.012, 0.004, -0.006]])


def _rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


@pytest.fixture(scope="module")
def rve8():
    return P.HfRve(8)


@pytest.mark.parametrize("tol,max_iter", [(1e-8, 30), (1e-9, 4), (1e-8, 3)])
def test_hf_trajectory_matches_oracle(rve8, tol, max_iter):
    """Identical Newton iteration counts (bisections included when max_iter=3
    forces them), sigma / C / snapshots within 1e-10."""
    opts = F.NewtonOptions(tol, max_iter, 6)
    g = rve8.trajectory(PATH, opts)
    o = O.Mesh(0, 8).hf_trajectory(DESK, PATH, tol=tol, max_iter=max_iter, max_bisections=6, snapshots=True)
    np.testing.assert_array_equal(g["iterations"], o["iterations"])
    assert _rel(g["sigma"], o["sigma"]) < 1e-10
    assert _rel(g["C"], o["C"]) < 1e-10
    assert _rel(g["snapshots"], o["snapshots"]) < 1e-9
    np.testing.assert_allclose(g["u_fluct_inf"], o["u_fluct_inf"], rtol=1e-9)
    assert g["snapshots"].shape == (len(PATH), rve8.n_dofs)


def test_hf_bisection_failure_is_solver_error(rve8):
    with pytest.raises(F.Fe2Error):
        rve8.trajectory(np.array([[0.2, -0.1, 0.3]]), F.NewtonOptions(1e-12, 1, 0))


def test_hf_deterministic(rve8):
    a = rve8.trajectory(PATH[:3])
    b = rve8.trajectory(PATH[:3])
    np.testing.assert_array_equal(a["sigma"], b["sigma"])
    np.testing.assert_array_equal(a["C"], b["C"])
    np.testing.assert_array_equal(a["snapshots"], b["snapshots"])


def test_band_ordering_is_narrow(rve8):
    """Reverse Cuthill-McKee keeps the free stiffness banded: half bandwidth
    well below the free DOF count (275 of 7,910 on default_cell(33))."""
    assert 0 < rve8.half_bandwidth < rve8.n_free // 3


def test_batched_trajectories_equal_serial_and_isolate_failures(rve8):
    """fe2_hf_trajectories: concurrent workers give bit-identical results to
    one-by-one fe2_hf_trajectory; a failing trajectory reports its error code
    and does not disturb the others."""
    rng = np.random.default_rng(3)
    T = 7
    ends = rng.standard_normal((T, 3))
    ends *= 0.015 / np.linalg.norm(ends, axis=1, keepdims=True)
    paths = np.stack([P.monotonic_path(e, 5) for e in ends])
    paths[4] = np.nan  # a NaN strain path: no Newton step converges (solver error)
    opts = F.NewtonOptions(1e-8, 30, 2)
    b = rve8.trajectories(paths, opts)
    assert b["status"][4] == 1 + 4 and (np.delete(b["status"], 4) == 0).all()
    for t in range(T):
        if t == 4:
            continue
        s = rve8.trajectory(paths[t], opts)
        for key in ("sigma", "C", "iterations", "snapshots", "res_last"):
            np.testing.assert_array_equal(b[key][t], s[key])


def test_batched_trajectories_match_oracle(rve8):
    """The POD training batch against the oracle's run_trajectory, per trajectory."""
    rng = np.random.default_rng(5)
    ends = rng.standard_normal((4, 3))
    ends *= 0.02 / np.linalg.norm(ends, axis=1, keepdims=True)
    paths = np.stack([P.monotonic_path(e, 6) for e in ends])
    b = rve8.trajectories(paths)
    assert (b["status"] == 0).all()
    for t in range(len(paths)):
        o = O.Mesh(0, 8).hf_trajectory(DESK, paths[t], snapshots=True)
        np.testing.assert_array_equal(b["iterations"][t], o["iterations"])
        assert _rel(b["sigma"][t], o["sigma"]) < 1e-10
        assert _rel(b["C"][t], o["C"]) < 1e-10
        assert _rel(b["snapshots"][t], o["snapshots"]) < 1e-9


def test_elastic_modes_match_oracle(rve8):
    g = rve8.elastic_modes()
    o = PO.elastic_modes(O.Mesh(0, 8), DESK)
    assert len(g) == 3
    np.testing.assert_allclose(g, o, atol=1e-9)
    np.testing.assert_allclose(g @ g.T, np.eye(3), atol=1e-12)


def _write_mesh(mesh, path):
    with open(path, "w") as f:
        f.write(f"fe2rom-mesh 1\nnodes {mesh.n_nodes}\n")
        for i, (x, y) in enumerate(mesh.xy):
            f.write(f"{i} {x:.17g} {y:.17g}\n")
        f.write(f"elements {mesh.n_elements}\n")
        for e in range(mesh.n_elements):
            f.write(f"{e} {mesh.mat[e]} " + " ".join(str(v) for v in mesh.conn[e]) + "\n")


def test_homogeneous_rve_exact(tmp_path):
    """homogeneous RVE -> zero fluctuation, Σ = C_e E,
    C_hom = C_e, and no elastic mode."""
    mesh = O.Mesh(geometry=1, subdivisions=4)
    _write_mesh(mesh, tmp_path / "h.mesh")
    rve = P.HfRve(materials=[F.ElasticParams(2.0, 0.25)] * 2, mesh_file=tmp_path / "h.mesh")
    E = np.array([[0.01, -0.004, 0.006]])
    r = rve.trajectory(E)
    lam, mu = 2.0 * 0.25 / (1.25 * 0.5), 1.0 / 1.25
    Ce = np.array([[lam + 2 * mu, lam, 0], [lam, lam + 2 * mu, 0], [0, 0, mu]])
    np.testing.assert_allclose(r["sigma"][0], Ce @ E[0], rtol=1e-10)
    np.testing.assert_allclose(r["C"][0], Ce, atol=1e-10 * Ce.max())
    assert r["u_fluct_inf"][0] < 1e-12
    assert len(rve.elastic_modes()) == 0


def _training(rve, n_traj=6, n_steps=8, seed=0):
    rng = np.random.default_rng(seed)
    ends = rng.standard_normal((n_traj, 3))
    ends *= 0.02 / np.linalg.norm(ends, axis=1, keepdims=True)
    return P.collect_snapshots(rve, ends, n_steps)


def test_pod_matches_numpy_oracle(rve8):
    X, meta = _training(rve8)
    assert X.shape[0] == len(meta) == 48
    Em = rve8.elastic_modes()
    V, s, mx = P.pod_basis(X, 12, Em)
    Vo, so, mxo = PO.pod(X, 12, Em)
    assert mx == mxo
    np.testing.assert_allclose(V @ V.T, np.eye(12), atol=1e-12)
    np.testing.assert_allclose(s[:12], so[:12], rtol=1e-10)
    # modes with well-separated singular values agree (sign fixed by convention)
    for j in range(3, 12):
        i = j - 3
        gap = min(abs(so[i] - so[i - 1]) if i else np.inf, abs(so[i] - so[i + 1]))
        if gap > 1e-3 * so[0]:
            np.testing.assert_allclose(V[j], Vo[j], atol=1e-8)
    assert P.max_usable_modes(X[:2], Em) == 3  # first steps are elastic: no mode beyond the elastic span
    with pytest.raises(F.Fe2Error):
        P.pod_basis(X[5:7], 6, Em)  # two plastic columns: 3 + rank 2 < 6
    assert P.max_usable_modes(X[5:7], Em) == 5


def test_rom_converges_to_hf():
    """hyper-ROM models (full rule) on POD bases of growing
    size (30 monotonic training trajectories, 10 steps, |E| = 0.025) approach
    the HF response on unseen paths: error non-increasing (within noise) and
    below 1% with enough modes (tools/rom_conv_probe.py has the sweep)."""
    rve = P.HfRve(12)
    rng = np.random.default_rng(1)
    ends = rng.standard_normal((30, 3))
    ends *= 0.025 / np.linalg.norm(ends, axis=1, keepdims=True)
    X, _ = P.collect_snapshots(rve, ends, 10)
    Em = rve.elastic_modes()
    for t in (np.array([0.012, -0.006, 0.010]), np.array([0.02, 0.0, 0.0]), np.array([-0.01, 0.015, -0.005])):
        path = np.stack([t * k / 10 for k in range(1, 11)])
        hf = rve.trajectory(path, snapshots=False)["sigma"]
        errs = []
        for n in (3, 6, 12, 24, 32):
            V, s, _ = P.pod_basis(X, n, Em)
            eng = F.HyperRomEngine.from_model(F.HyperRomModel(12, K=0, basis=V))
            eng.alloc_points(1)
            sig = np.stack([eng.solve_increment(path[k][None])["sigma"][0] for k in range(len(path))])
            errs.append(np.linalg.norm(sig - hf) / np.linalg.norm(hf))
        assert errs[-1] < 0.01, errs
        for a, b in zip(errs, errs[1:]):
            assert b <= a * 1.05, errs
