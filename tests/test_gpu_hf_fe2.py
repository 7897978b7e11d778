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


def _grid_mesh(path, m=3):
    """A small heterogeneous RVE in the reference's mesh format (write_mesh,
    mesh.hpp:413-431): m x m squares of two Tri6 each, the centre square an
    inclusion (material 1); (2m+1)^2 nodes, 2 (2m-1)^2 free DOFs (linear BC)."""
    k = 2 * m + 1
    xy = [(i / (k - 1), j / (k - 1)) for j in range(k) for i in range(k)]
    nid = lambda i, j: j * k + i  # noqa: E731
    els = []
    for bj in range(m):
        for bi in range(m):
            i0, j0 = 2 * bi, 2 * bj
            c00, c10, c11, c01 = nid(i0, j0), nid(i0 + 2, j0), nid(i0 + 2, j0 + 2), nid(i0, j0 + 2)
            mat = 1 if (bi, bj) == (m // 2, m // 2) else 0
            els.append((mat, c00, c10, c11, nid(i0 + 1, j0), nid(i0 + 2, j0 + 1), nid(i0 + 1, j0 + 1)))
            els.append((mat, c00, c11, c01, nid(i0 + 1, j0 + 1), nid(i0 + 1, j0 + 2), nid(i0, j0 + 1)))
    with open(path, "w") as f:
        f.write(f"fe2rom-mesh 1\nnodes {len(xy)}\n")
        for i, (x, y) in enumerate(xy):
            f.write(f"{i} {x:.17g} {y:.17g}\n")
        f.write(f"elements {len(els)}\n")
        for e, (mat, *nodes) in enumerate(els):
            f.write(f"{e} {mat} " + " ".join(map(str, nodes)) + "\n")
    return xy


def test_hf_monolithic_iterations_equal_full_basis_hyper_rom(tmp_path):
    """HF_monolithic (fe2_hf_mono_*) is the hyper-ROM monolithic algebra on the
    full field: with Φ = identity on the free DOFs and the full quadrature, the
    hyper-ROM engine's monolithic iterates (fe2_hrom_mono_*) are the same
    (SPEC.md:591 equivalence) — Σ~ and C of every iteration within 1e-9, over
    steps with moving macro strains and commits. (The mesh's half bandwidth, 19,
    is below the 32-column panels: the narrow-band path of the band solver.)"""
    mesh = tmp_path / "grid3.txt"
    xy = _grid_mesh(mesh, 3)
    on_b = [x in (0.0, 1.0) or y in (0.0, 1.0) for x, y in xy]
    free = [2 * v + c for v in range(len(xy)) if not on_b[v] for c in (0, 1)]
    V = np.zeros((len(free), 2 * len(xy)))
    for r, d in enumerate(free):
        V[r, d] = 1.0
    md = F.HyperRomModel(mesh_file=str(mesh), K=0, basis=V)
    assert md.n == len(free) == 50
    eng = F.HyperRomEngine.from_model(md)
    hf = P.HfRve(mesh_file=str(mesh))
    assert hf.n_free == md.n
    Pn = 3
    eng.alloc_points(Pn)
    hf.alloc_points(Pn)
    base = np.array([[0.012, -0.004, 0.008], [-0.006, 0.010, 0.004], [0.004, 0.003, -0.012]])
    n_plastic = 0
    for step in range(3):
        eng.mono_begin()
        hf.mono_begin()
        for it in range(3):
            E = base * (step + 1) * (1.0 + 0.05 * it)  # the macro iterate moves within a step
            g = eng.mono_iterate(E)
            h = hf.mono_iterate(E)
            assert (g["status"] == 0).all() and (h["status"] == 0).all()
            n_plastic += int(g["plastic_count"].sum())
            for key in ("sigma", "C"):
                a, b = h[key].reshape(Pn, -1), g[key].reshape(Pn, -1)
                assert np.abs(a - b).max() < 1e-9 * np.abs(b).max(), (step, it, key)
            # (rel_res is method-specific: |r| over max(|r_first|, |reactions|) for the full field as
            # micro_newton, over max(|r_first|, |Σ_raw|) for the reduced path, DESIGN §2 decision 4)
            assert (h["rel_res"] <= 1.0 + 1e-12).all()
        eng.mono_commit()
        hf.mono_commit()
    assert n_plastic > 0


def test_hf_monolithic_driver_same_fixed_point_as_nested(rve8):
    """SPEC.md:480 example: the HF_monolithic FE² beam converges to the
    HF_nested fixed point (R within 1e-5 relative, U_res within 1e-4 Ū)."""
    # (steps small enough that neither scheme bisects: a bisected sub-step is a
    # different plastic loading path, e.g. 5e-4 in R at n_load = 4)
    cfg = F.MacroConfig(u_max=0.2, n_load=8, max_unload=16)
    nested = F.solve_program(cfg, rve8)
    cfg_m = F.MacroConfig(u_max=0.2, n_load=8, max_unload=16, scheme="monolithic")
    mono = F.solve_program(cfg_m, P.HfRve(8))
    assert len(mono["U"]) == len(nested["U"])
    np.testing.assert_allclose(mono["U"], nested["U"], rtol=0, atol=1e-12)
    assert np.abs(mono["R"] - nested["R"]).max() < 1e-5 * np.abs(nested["R"]).max()
    assert abs(mono["U_residual"] - nested["U_residual"]) < 1e-4 * cfg.u_max
    assert nested["U_residual"] > 0
