"""Empirical Cubature Method (SPEC.md:333-369
hyper.ecm_select): the host selection against its numpy restatement and the
SPEC examples / invariants (constant-only basis, full rule, volume
exactness, positive weights, monotone residual)."""
import numpy as np
import pytest

import ecm_oracle as EO
import paper_2306_02687_b200.ecm as E


def test_constant_only_basis_single_point():
    w = np.random.default_rng(0).uniform(0.5, 1.5, 300) / 300
    ids, wt, res = E.ecm_select(np.zeros((300, 0)), w, 10)
    assert len(ids) == 1 and abs(wt[0] - w.sum()) < 1e-12 * w.sum() and res < 1e-14


def test_full_rule_is_feasible():
    m = 40
    w = np.random.default_rng(1).uniform(0.5, 1.5, m)
    ids, wt, res = E.ecm_select(np.eye(m), w, m + 1, 1e-14)
    np.testing.assert_array_equal(ids, np.arange(m))
    np.testing.assert_allclose(wt, w, rtol=1e-12)
    assert res < 1e-13


@pytest.mark.parametrize("m,k,seed", [(500, 20, 0), (2000, 60, 1), (300, 30, 2)])
def test_selection_matches_numpy_restatement(m, k, seed):
    rng = np.random.default_rng(seed)
    # smooth-ish integrands: orthonormalised polynomials of random point coordinates
    x = rng.uniform(size=(m, 2))
    F = np.stack([x[:, 0] ** i * x[:, 1] ** j for i in range(8) for j in range(8)][:k], axis=1)
    U = np.linalg.qr(F)[0]
    w = rng.uniform(0.5, 1.5, m) / m
    ids, wt, res = E.ecm_select(U, w, k + 1, 1e-12)
    ido, wo, reso = EO.ecm_select(U, w, k + 1, 1e-12)
    np.testing.assert_array_equal(ids, ido)
    np.testing.assert_allclose(wt, wo, rtol=1e-8)
    assert (wt > 0).all() and len(set(ids.tolist())) == len(ids)
    assert abs(wt.sum() - w.sum()) <= 1e-8 * w.sum()  # volume exactness
    assert res <= 1e-10
    # exact reproduction of every mode's integral
    np.testing.assert_allclose(U[ids].T @ wt, U.T @ w, atol=1e-10 * np.abs(U.T @ w).max())


def test_residual_monotone_in_target():
    rng = np.random.default_rng(3)
    m, k = 800, 40
    x = rng.uniform(size=(m, 2))
    F = np.stack([np.cos(i * x[:, 0] + j * x[:, 1]) for i in range(7) for j in range(7)][:k], axis=1)
    U = np.linalg.qr(F)[0]
    w = np.full(m, 1.0 / m)
    res = [E.ecm_select(U, w, t, 0.0)[2] for t in (5, 10, 20, 30, 41)]
    assert all(b <= a * (1 + 1e-12) for a, b in zip(res, res[1:]))
    assert res[-1] < 1e-10


def test_rule_text_round_trip(tmp_path):
    rng = np.random.default_rng(4)
    ids = np.sort(rng.choice(6075, 87, replace=False)).astype(np.int32)
    w = rng.uniform(1e-5, 1e-3, 87)
    E.save_rule(tmp_path / "rule.txt", ids, w)
    i2, w2 = E.load_rule(tmp_path / "rule.txt")
    np.testing.assert_array_equal(i2, ids)
    np.testing.assert_array_equal(w2, w)
