"""GPU parity at the BASELINE configs' real sizes (VERDICT r01 "next" #1).

north_star bar: Newton iteration counts and per-(point, cubature point) plastic/elastic
flags identical to the CPU oracle, macro stress and tangent within 1e-10 relative (fp64).
- config 1: ALL 65,536 points x 50 increments (flags of every commit, compared in chunks);
- config 2: 1,024 points x all 30 increments (finite strain; oracle parity-unpinned model);
- config 3: n = 64, K = 2,000 (the multi-GPU config's model) on 128 points x 20 increments;
- config 4: the grid corners n x K = 128 x 4,000, 64 x 4,000, 8 x 4,000 (ring kernel).
"""
import os

import numpy as np
import pytest

import paper_2306_02687_b200 as F
import pyoracle as O

from test_gpu_parity import REL, path_rel_err, rel_err

pytestmark = pytest.mark.gpu
THREADS = os.cpu_count() or 8


def run_gpu_flags(m, E, fs=False):
    """All increments on the device; per increment the outputs and the packed plastic flags."""
    eng = F.HyperRomEngine.from_model(m, finite_strain=fs)
    P, n_incr = E.shape[:2]
    eng.alloc_points(P, keep_flags=True)
    outs, flags = [], []
    for k in range(n_incr):
        outs.append(eng.solve_increment(np.ascontiguousarray(E[:, k])))
        flags.append(np.packbits(eng.read_state(flags=True)[2], axis=1))
    g = {key: np.stack([o[key] for o in outs], axis=1) for key in outs[0]}
    return eng, g, np.stack(flags, axis=1)  # [P, incr, ceil(K/8)]


def check_chunk(g, flags_packed, o, sl, K, fs=False):
    np.testing.assert_array_equal(g["status"][sl], o["status"])
    np.testing.assert_array_equal(g["iters"][sl], o["iters"])
    np.testing.assert_array_equal(g["plastic_count"][sl], o["plastic_count"])
    gf = np.unpackbits(flags_packed[sl], axis=2, count=K)
    np.testing.assert_array_equal(gf, o["plastic_flags"])
    o_s, o_c, c_dim = ("P", "A", 16) if fs else ("sigma", "C", 9)  # device: sigma = P_M, C = A_M
    assert path_rel_err(g["sigma"][sl], o[o_s]).max() < REL
    assert rel_err(g["C"][sl].reshape(-1, c_dim), o[o_c].reshape(-1, c_dim)).max() < REL


def test_config1_all_points_all_increments():
    m = F.HyperRomModel(33, 24, 400, 0)
    P, n_incr = 65536, 50
    E = F.make_paths(1, 0, P, n_incr)
    _, g, fl = run_gpu_flags(m, E)
    assert (g["status"] == 0).all()
    orc = O.Hrom(m.G, m.w, m.mat, m.materials, m.volume)
    chunk = 4096
    n_plastic = 0
    for p0 in range(0, P, chunk):
        sl = slice(p0, p0 + chunk)
        o = orc.run(np.ascontiguousarray(E[sl]), threads=THREADS, flags=True)
        check_chunk(g, fl, o, sl, m.K)
        n_plastic += int(o["plastic_flags"].sum())
    assert n_plastic > 0


def test_config2_finite_strain_1024_points_all_increments():
    m = F.HyperRomModel(33, 32, 600, 0)
    P, n_incr = 1024, 30
    H = F.make_paths(2, 0, P, n_incr)
    _, g, fl = run_gpu_flags(m, H, fs=True)
    assert (g["status"] == 0).all()
    o = O.HromFs(m.G4, m.w, m.mat, m.materials, m.volume).run(H, threads=THREADS, flags=True)
    check_chunk(g, fl, o, slice(0, P), m.K, fs=True)
    assert o["plastic_flags"].sum() > 0


def test_config3_model_real_size():
    """n = 64, K = 2,000 (1,460 J2 points), config-0 paths, 20 increments."""
    m = F.HyperRomModel(33, 64, 2000, 0)
    P, n_incr = 128, 20
    E = F.make_paths(0, 0, P, n_incr)
    eng, g, fl = run_gpu_flags(m, E)
    o = O.Hrom(m.G, m.w, m.mat, m.materials, m.volume).run(E, threads=THREADS, flags=True, final_state=True)
    assert (o["status"] == 0).all()
    check_chunk(g, fl, o, slice(0, P), m.K)
    alpha, state, _ = eng.read_state()
    np.testing.assert_allclose(alpha, o["alpha"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(state, o["state"], rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("n,K,P", [(128, 4000, 32), (64, 4000, 64), (8, 4000, 256), (16, 4000, 128), (24, 1500, 128)])
def test_config4_corners(n, K, P):
    """Roofline-sweep corners: config-0 generator, 5 increments. n = 16 / 24 with an operator too
    large for shared memory run the 12-warp ring variant of k_increment."""
    m = F.HyperRomModel(33, n, K, 0)
    E = F.make_paths(0, 0, P, 5)
    _, g, fl = run_gpu_flags(m, E)
    o = O.Hrom(m.G, m.w, m.mat, m.materials, m.volume).run(E, threads=THREADS, flags=True)
    assert (o["status"] == 0).all()
    check_chunk(g, fl, o, slice(0, P), m.K)
