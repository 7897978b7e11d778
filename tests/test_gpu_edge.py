"""Edge cases of the device path against the oracle: one macro point, one
mode, a model without J2 points (all elastic: no history at all), one
without elastic points, the first CTA-per-point size (n = 33), and the
finite-strain path without J2 points."""
import numpy as np
import pytest

import paper_2306_02687_b200 as F
import pyoracle as O

pytestmark = pytest.mark.gpu


def run_both(G, w, mat, mats, vol, E, finite=False):
    eng = F.HyperRomEngine(G, w, mat, mats, vol)
    eng.alloc_points(E.shape[0], keep_flags=True)
    outs = [eng.solve_increment(E[:, k]) for k in range(E.shape[1])]
    g = {k: np.stack([o[k] for o in outs], axis=1) for k in outs[0]}
    orc = (O.HromFs if finite else O.Hrom)(G, w, mat, mats, vol)
    o = orc.run(E, threads=8)
    return g, o


def check(g, o, finite=False):
    np.testing.assert_array_equal(g["status"], o["status"])
    np.testing.assert_array_equal(g["iters"], o["iters"])
    np.testing.assert_array_equal(g["plastic_count"], o["plastic_count"])
    so = o["P"] if finite else o["sigma"]
    scale = np.abs(so).max()
    assert np.abs(g["sigma"] - so).max() <= 1e-10 * scale
    Co = o["A"] if finite else o["C"]
    assert np.abs(g["C"] - Co).max() <= 1e-10 * np.abs(Co).max()


def test_single_point_and_single_mode():
    m = F.HyperRomModel(33, 1, 50, 3)
    E = F.make_paths(0, 0, 1, 12)
    check(*run_both(m.G, m.w, m.mat, m.materials, m.volume, E))


def test_all_elastic_model_has_no_history():
    m = F.HyperRomModel(33, 12, 200, 0)
    mat = np.ones_like(m.mat)  # every cubature point in the elastic inclusion material
    E = F.make_paths(0, 0, 64, 8)
    g, o = run_both(m.G, m.w, mat, m.materials, m.volume, E)
    check(g, o)
    assert (o["plastic_count"] == 0).all() and (g["iters"] <= 1).all()


def test_all_j2_model():
    m = F.HyperRomModel(33, 16, 300, 1)
    mat = np.zeros_like(m.mat)
    E = F.make_paths(1, 0, 96, 20)
    check(*run_both(m.G, m.w, mat, m.materials, m.volume, E))


def test_first_cta_per_point_size():
    m = F.HyperRomModel(33, 33, 300, 2)
    E = F.make_paths(0, 0, 24, 6)
    check(*run_both(m.G, m.w, m.mat, m.materials, m.volume, E))


def test_finite_strain_without_j2_points():
    m = F.HyperRomModel(12, 8, 60, 1)
    mat = np.ones_like(m.mat)
    H = F.make_paths(2, 0, 32, 6)
    g, o = run_both(m.G4, m.w, mat, m.materials, m.volume, H, finite=True)
    check(g, o, finite=True)


def test_empty_and_oversized_batches_fail_cleanly():
    """P = 0 is a config error; a batch beyond HBM fails with ErrorCode::numeric
    (device allocation) and the handle then serves a normal batch."""
    m = F.HyperRomModel(33, 12, 200, 0)
    eng = F.HyperRomEngine.from_model(m)
    with pytest.raises(F.Fe2Error) as e:
        eng.alloc_points(0)
    assert e.value.kind == "config"
    with pytest.raises(F.Fe2Error) as e:
        eng.alloc_points((1 << 31) - 1)  # ~0.5 PB of history
    assert e.value.kind == "numeric" and "allocation" in str(e.value)
    E = F.make_paths(0, 0, 16, 4)
    eng.alloc_points(16)
    outs = [eng.solve_increment(E[:, k]) for k in range(4)]
    o = O.Hrom(m.G, m.w, m.mat, m.materials, m.volume).run(E, threads=4)
    np.testing.assert_array_equal(np.stack([x["iters"] for x in outs], 1), o["iters"])
