"""GPU parity of the finite-strain (Biot stress) path, BASELINE config 2,
against the CPU oracle's fs_* restatement on identical seeded inputs.
PARITY UNPINNED: the reference has no finite-strain code; the oracle is
anchored by tests/test_oracle_fs.py (FD tangents, objectivity, small-strain
limit to the pinned small-strain oracle). Same bar as the small-strain path:
identical Newton iteration counts and plastic flags, P_M and A_M within
1e-10 relative (fp64)."""
import numpy as np
import pytest

import paper_2306_02687_b200 as F
import pyoracle as O

pytestmark = pytest.mark.gpu

REL = 1e-10


def rel_err(a, b):
    a, b = np.asarray(a), np.asarray(b)
    num = np.linalg.norm((a - b).reshape(a.shape[0], -1), axis=1)
    den = np.linalg.norm(b.reshape(b.shape[0], -1), axis=1)
    return num / np.maximum(den, 1e-300)


def engine(m, P, keep_flags=False):
    eng = F.HyperRomEngine.from_model(m, finite_strain=True)
    eng.alloc_points(P, keep_flags=keep_flags)
    return eng


def oracle(m):
    return O.HromFs(m.G4, m.w, m.mat, m.materials, m.volume)


def run_gpu(eng, H, opts=None, flags=False):
    outs, fl = [], []
    for k in range(H.shape[1]):
        outs.append(eng.solve_increment(H[:, k], opts))
        if flags:
            fl.append(eng.read_state(flags=True)[2])
    g = {k: np.stack([o[k] for o in outs], axis=1) for k in outs[0]}
    if flags:
        g["flags"] = np.stack(fl, axis=1)
    return g


def check_parity(g, o, P, k):
    assert (o["status"] == 0).all() and (g["status"] == 0).all()
    np.testing.assert_array_equal(g["iters"], o["iters"])
    np.testing.assert_array_equal(g["plastic_count"], o["plastic_count"])
    es = rel_err(g["sigma"].reshape(P * k, 4), o["P"].reshape(P * k, 4))
    ea = rel_err(g["C"].reshape(P * k, 16), o["A"].reshape(P * k, 16))
    assert es.max() < REL, es.max()
    assert ea.max() < REL, ea.max()


def test_fs_assembly_matches_oracle():
    m = F.HyperRomModel(33, 32, 600, 0)
    H = F.make_paths(2, 0, 4, 30)
    eng = engine(m, 4)
    orc = oracle(m)
    # history: commit a few increments on the GPU and in the oracle
    for k in range(12):
        eng.solve_increment(H[:, k])
    o_run = orc.run(H[:1, :12], final_state=True)
    alpha_g, state_g, _ = eng.read_state()
    np.testing.assert_allclose(alpha_g[0], o_run["alpha"][0], rtol=1e-9, atol=1e-13)
    st = o_run["state"][0]
    assert (st[:, 4] > 0).any()
    rng = np.random.default_rng(5)
    for trial in range(3):
        alpha = o_run["alpha"][0] + rng.normal(scale=0.002, size=m.n)
        Hv = H[0, 12 + trial] * (1.0 + 0.1 * trial)
        g = eng.fs_assemble_point(0, alpha, Hv)
        o = orc.assemble(alpha, Hv, st)
        for key in ("r", "Kaa", "KaF", "KFa", "C_FF", "P_raw"):
            err = np.linalg.norm(g[key] - o[key]) / np.linalg.norm(o[key])
            assert err < 1e-12, (key, err)


def test_fs_small_model_trajectory_parity():
    m = F.HyperRomModel(12, 8, 60, 1)
    H = F.make_paths(2, 3, 96, 12)
    eng = engine(m, 96, keep_flags=True)
    g = run_gpu(eng, H, flags=True)
    o = oracle(m).run(H, threads=8, flags=True, final_state=True)
    check_parity(g, o, 96, 12)
    np.testing.assert_array_equal(g["flags"], o["plastic_flags"])
    assert o["plastic_count"].max() > 0
    alpha, state, _ = eng.read_state()
    np.testing.assert_allclose(alpha, o["alpha"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(state, o["state"], rtol=1e-9, atol=1e-12)


def test_fs_config2_subset_parity():
    """BASELINE config 2 model (n = 32, K = 600) and path generator, 30
    increments, on a point subset the oracle finishes in seconds."""
    m = F.HyperRomModel(33, 32, 600, 0)
    P = 96
    H = F.make_paths(2, 0, P, 30)
    eng = engine(m, P, keep_flags=True)
    g = run_gpu(eng, H, flags=True)
    o = oracle(m).run(H, threads=16, flags=True)
    check_parity(g, o, P, 30)
    np.testing.assert_array_equal(g["flags"], o["plastic_flags"])
    assert (o["plastic_count"] > 0).mean() > 0.5


@pytest.mark.parametrize("n,K", [(16, 300), (24, 400)])
def test_fs_widths_trajectory_parity(n, K):
    m = F.HyperRomModel(33, n, K, 2)
    H = F.make_paths(2, 1, 48, 10)
    g = run_gpu(engine(m, 48), H)
    o = oracle(m).run(H, threads=8)
    check_parity(g, o, 48, 10)


def test_fs_bisection_and_failure_parity():
    m = F.HyperRomModel(12, 8, 60, 1)
    H = F.make_paths(2, 0, 32, 2)
    opts = F.NewtonOptions(max_iter=2, max_bisections=8)
    g = run_gpu(engine(m, 32), H, opts)
    o = oracle(m).run(H, max_iter=2, max_bisections=8)
    np.testing.assert_array_equal(g["status"], o["status"])
    np.testing.assert_array_equal(g["iters"], o["iters"])
    ok = o["status"] == 0
    assert (o["bisections"] > 0).any()
    assert rel_err(g["sigma"][ok], o["P"][ok]).max() < REL
    # failure: NaN outputs and the solver code, on the same points
    opts = F.NewtonOptions(max_iter=1, max_bisections=0)
    g = run_gpu(engine(m, 32), H, opts)
    o = oracle(m).run(H, max_iter=1, max_bisections=0)
    np.testing.assert_array_equal(g["status"], o["status"])
    bad = o["status"] != 0
    assert bad.any() and np.isnan(g["sigma"][bad]).all() and np.isnan(g["C"][bad]).all()


def test_fs_large_batch_properties():
    """Full config-2 point count on the device (262,144 points) for two
    increments: all converge, and sampled points equal the oracle."""
    m = F.HyperRomModel(33, 32, 600, 0)
    P = 262144
    H = F.make_paths(2, 0, P, 30)
    eng = engine(m, P)
    g = run_gpu(eng, np.ascontiguousarray(H[:, :2]))
    assert (g["status"] == 0).all()
    idx = np.array([0, 1, 77, 4095, 100000, P - 1])
    o = oracle(m).run(np.ascontiguousarray(H[idx, :2]), threads=6)
    np.testing.assert_array_equal(g["iters"][idx], o["iters"])
    assert rel_err(g["sigma"][idx].reshape(-1, 4), o["P"].reshape(-1, 4)).max() < REL
    assert rel_err(g["C"][idx].reshape(-1, 16), o["A"].reshape(-1, 16)).max() < REL
