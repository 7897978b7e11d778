"""Offline ECM pipeline on the device engine: integrand
snapshots from full-rule training trajectories, SVD, ECM selection; the
hyper-ROM with the selected rule reproduces the full-rule ROM's macro
stress, and the rule runs through the hot path with exact parity against
the oracle."""
import numpy as np
import pytest

import paper_2306_02687_b200 as F
import paper_2306_02687_b200.ecm as E
import pyoracle as O

pytestmark = pytest.mark.gpu


def test_ecm_rule_reproduces_full_rule_rom():
    full = F.HyperRomModel(33, 8, 0, 0)  # all 6,075 integration points, their own weights
    assert full.K == 6075 and abs(full.w.sum() - full.volume) < 1e-12
    train = np.concatenate([F.make_paths(0, 0, 16, 10), F.make_paths(1, 0, 16, 50)[:, ::5]], axis=0)
    ids, w, res, k = E.build_rule(full, train, m_target=300, tol=1e-10, svd_tol=1e-4)
    assert len(ids) <= k + 1 and (w > 0).all() and res < 1e-8
    assert abs(w.sum() - full.volume) < 1e-8 * full.volume
    test = F.make_paths(0, 7, 64, 10, p0=1000)
    ref = F.HyperRomEngine.from_model(full)
    ref.alloc_points(64)
    hyp = F.HyperRomEngine(full.G[ids], w, full.mat[ids], full.materials, full.volume)
    hyp.alloc_points(64)
    worst = 0.0
    for kk in range(10):
        a, b = ref.solve_increment(test[:, kk]), hyp.solve_increment(test[:, kk])
        assert (a["status"] == 0).all() and (b["status"] == 0).all()
        worst = max(worst, np.abs(b["sigma"] - a["sigma"]).max() / np.abs(a["sigma"]).max())
    assert worst < 1e-3, worst
    # the ECM rule is an ordinary hot-path input: exact parity with the oracle
    orc = O.Hrom(full.G[ids], w, full.mat[ids], full.materials, full.volume)
    o = orc.run(test, threads=8)
    hyp.reset_points()
    g = [hyp.solve_increment(test[:, kk]) for kk in range(10)]
    np.testing.assert_array_equal(np.stack([x["iters"] for x in g], 1), o["iters"])
    sg = np.stack([x["sigma"] for x in g], 1)
    assert np.abs(sg - o["sigma"]).max() <= 1e-10 * np.abs(o["sigma"]).max()
