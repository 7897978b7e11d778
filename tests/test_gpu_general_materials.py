"""GPU parity of the hyper-ROM engine with iterative history materials:
power-law hardening (materials.hpp:216-244) and strain-hardening creep
(:246-292, the paper's Example 2 material) at the
cubature points of the matrix, elastic inclusions elsewhere.

The device runs the reference's safeguarded scalar Newton per cubature point
(general_return, device_common.cuh) inside k_increment / k_increment_big; a
creep sub-step integrates over PathStep::dt x its fraction (rve.hpp:466).
Bar (north_star): identical Newton iteration counts, status and per-(point,
cubature point) plastic flags, Σ / C_macro within 1e-10 relative."""
import os

import numpy as np
import pytest

import paper_2306_02687_b200 as F
import pyoracle as O

from test_gpu_full_configs import run_gpu_flags
from test_gpu_parity import REL, path_rel_err, rel_err

pytestmark = pytest.mark.gpu
THREADS = os.cpu_count() or 8

POWER = F.PowerLawParams(1.0, 0.3, 0.01, 0.1)
CREEP = F.CreepParams(1.0, 0.14, 22.09, 1.06, -0.56, 1.0)  # PAPER.md:124 (E = 1)
CREEP_FAST = F.CreepParams(1.0, 0.14, 0.02, 1.06, -0.56, 0.5)  # visibly relaxing
INCL = F.ElasticParams(10.0, 0.3)


def model(n, K, mats):
    m = F.HyperRomModel(33, n, K, 0)
    m.materials = list(mats)
    return m


def compare(m, E, opts=None):
    eng, g, fl = run_gpu_flags(m, E) if opts is None else run_gpu_opts(m, E, opts)
    kw = {} if opts is None else dict(tol=opts.tol, max_iter=opts.max_iter, max_bisections=opts.max_bisections)
    o = O.Hrom(m.G, m.w, m.mat, m.materials, m.volume).run(E, threads=THREADS, flags=True, **kw)
    np.testing.assert_array_equal(g["status"], o["status"])
    np.testing.assert_array_equal(g["iters"], o["iters"])
    ok = o["status"] == 0  # failed increments carry no response (run_trajectory throws)
    np.testing.assert_array_equal(g["plastic_count"][ok], o["plastic_count"][ok])
    gf = np.unpackbits(fl, axis=2, count=m.K)
    np.testing.assert_array_equal(gf[ok], o["plastic_flags"][ok])
    assert np.isnan(g["sigma"][~ok]).all() and np.isnan(g["C"][~ok]).all()
    if ok.any():
        okp = ok.all(axis=1)  # points whose whole trajectory succeeded: path-relative Σ error
        if okp.any():
            assert path_rel_err(g["sigma"][okp], o["sigma"][okp]).max() < REL
        assert rel_err(g["C"][ok].reshape(-1, 9), o["C"][ok].reshape(-1, 9)).max() < REL
    return g, o


def run_gpu_opts(m, E, opts):
    eng = F.HyperRomEngine.from_model(m)
    P, n_incr = E.shape[:2]
    eng.alloc_points(P, keep_flags=True)
    outs, flags = [], []
    for k in range(n_incr):
        outs.append(eng.solve_increment(np.ascontiguousarray(E[:, k]), opts))
        flags.append(np.packbits(eng.read_state(flags=True)[2], axis=1))
    g = {key: np.stack([o[key] for o in outs], axis=1) for key in outs[0]}
    return eng, g, np.stack(flags, axis=1)


@pytest.mark.parametrize("n,K,P,path", [(12, 200, 512, 0), (24, 400, 256, 1)])
def test_power_law_warp_kernel(n, K, P, path):
    m = model(n, K, [POWER, INCL])
    E = F.make_paths(path, 0, P, 20)
    g, o = compare(m, E)
    assert (o["status"] == 0).all()
    fl = o["plastic_flags"][:, :, m.mat == 0]
    assert 0.05 < fl.mean() < 0.95  # mixed elastic / plastic points


@pytest.mark.parametrize("mat", [CREEP, CREEP_FAST], ids=["paper", "fast"])
def test_creep_paper_sizes(mat):
    """n = 30 modes, K = 500 cubature points: the paper's Example 2 sizes."""
    m = model(30, 500, [mat, INCL])
    E = F.make_paths(1, 0, 128, 20)
    g, o = compare(m, E)
    assert (o["status"] == 0).all()
    assert o["plastic_flags"][:, :, m.mat == 0].mean() > 0.9  # creep flows wherever q > 0


@pytest.mark.parametrize("mat,path,tol,max_iter", [(CREEP_FAST, 1, 1e-4, 1), (POWER, 0, 1e-8, 2)],
                         ids=["creep", "power"])
def test_bisected_substeps(mat, path, tol, max_iter):
    """A small max_iter forces bisected sub-steps (rve.hpp:473-478); a creep
    sub-step integrates over its share of dt (:466). Some trajectories exhaust
    the bisections (status 1 + solver) and end there."""
    m = model(12, 200, [mat, INCL])
    E = F.make_paths(path, 0, 128, 10)
    g, o = compare(m, E, F.NewtonOptions(tol, max_iter, 4))
    assert o["bisections"].sum() > 50
    assert (o["status"] == 0).mean() > 0.5


@pytest.mark.parametrize("mat,n,K", [(POWER, 64, 1000), (CREEP_FAST, 64, 1000), (CREEP_FAST, 128, 1000),
                                     (POWER, 40, 600)], ids=["power64", "creep64", "creep128", "power40"])
def test_cta_kernel(mat, n, K):
    """n > 32: the CTA-per-point kernel (k_increment_big<NT, false, GEN>, its own unit)."""
    m = model(n, K, [mat, INCL])
    E = F.make_paths(0, 0, 16 if n > 64 else 32, 8)
    g, o = compare(m, E)
    assert (o["status"] == 0).all()


@pytest.mark.parametrize("n,K", [(12, 200), (64, 600)])
def test_material_failure_ends_trajectory(n, K):
    """dt = 0 makes every creep update fail (materials.hpp:249, ErrorCode::material):
    status 1 + material on the first increment and on every later one, no response."""
    m = model(n, K, [F.CreepParams(1.0, 0.14, 22.09, 1.06, -0.56, 0.0), INCL])
    E = F.make_paths(0, 0, 16, 3)
    g, o = compare(m, E)
    assert (o["status"] == 1 + 3).all()
    assert np.isnan(g["sigma"]).all()


def test_monolithic_iteration_rejects_iterative_materials():
    m = model(12, 200, [CREEP, INCL])
    eng = F.HyperRomEngine.from_model(m)
    eng.alloc_points(4)
    with pytest.raises(F.Fe2Error) as e:
        eng.mono_begin()
    assert e.value.code == 1
