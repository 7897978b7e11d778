"""The product's offline stage (seeded hyper-ROM model and macro paths, C++ in
libfe2rom_gpu.so, host only) against the oracle's independent restatement:
bit-for-bit equal G_q, weights, cubature ids, material ids, volume, paths."""
import numpy as np
import pytest

import paper_2306_02687_b200 as F
import pyoracle as O


@pytest.mark.parametrize("sub,n,K,seed", [(33, 12, 200, 0), (33, 24, 400, 0), (8, 6, 50, 7), (12, 16, 300, 3)])
def test_model_bitwise_equal_to_oracle(sub, n, K, seed):
    m = F.HyperRomModel(sub, n, K, seed)
    o = O.Model(sub, n, K, seed)
    assert (m.n, m.K, m.n_free) == (o.n, o.K, o.n_free)
    assert m.volume == o.volume
    assert np.array_equal(m.ip, o.ip) and np.array_equal(m.mat, o.mat)
    assert np.array_equal(m.w, o.w)
    assert np.array_equal(m.G, o.G)


def test_model_properties():
    o = O.Model(33, 24, 400, 0)
    # Φ orthonormal (Householder thin Q) on the free DOFs
    assert np.abs(o.phi.T @ o.phi - np.eye(24)).max() < 1e-13
    # K distinct integration points, weights U[0.5, 1.5] area / K
    assert len(set(o.ip.tolist())) == 400
    assert o.w.min() >= 0.5 * o.volume / 400 and o.w.max() < 1.5 * o.volume / 400
    assert set(np.unique(o.mat).tolist()) == {0, 1}
    # G_q = B_q Φ[dofs(el(q))]: recompute a few rows from the mesh B matrices
    mesh = O.Mesh(0, 33)
    free = np.ones(2 * mesh.n_nodes, bool)
    for i, (x, y) in enumerate(mesh.xy):
        if min(abs(x), abs(x - 1), abs(y), abs(y - 1)) < 1e-12:
            free[2 * i] = free[2 * i + 1] = False
    fidx = np.cumsum(free) - 1
    for q in (0, 17, 399):
        B, w, e = mesh.ip(int(o.ip[q]))
        dofs = np.array([2 * nd + c for nd in mesh.conn[e] for c in (0, 1)])
        Phi_el = np.where(free[dofs, None], o.phi[np.clip(fidx[dofs], 0, None)], 0.0)
        np.testing.assert_allclose(B @ Phi_el, o.G[q], rtol=0, atol=1e-13)


@pytest.mark.parametrize("kind,n_incr", [(0, 20), (1, 50)])
def test_paths_bitwise_and_shape(kind, n_incr):
    E = F.make_paths(kind, 0, 300, n_incr)
    assert np.array_equal(E, O.paths(kind, 0, 300, n_incr))
    # per-point streams keyed by the global point index: any shard equals the slice
    assert np.array_equal(F.make_paths(kind, 0, 100, n_incr, p0=150), E[150:250])
    if kind == 0:  # uniaxial 0.05 s rotated by theta: E11 + E22 = 0.05 s in [0.025, 0.075]
        tr = E[:, -1, 0] + E[:, -1, 1]
        assert tr.min() >= 0.025 - 1e-15 and tr.max() <= 0.075 + 1e-15
        np.testing.assert_allclose(E[:, 9], 0.5 * E[:, 19], rtol=1e-14)
    else:  # reversal: peak at the half, back to zero at the end, E22 = 0
        assert np.abs(E[:, -1]).max() == 0.0 and np.abs(E[:, :, 1]).max() == 0.0
        assert np.abs(E[:, 24, 0]).max() <= 0.03 and np.abs(E[:, 24, 2]).max() <= 0.04
        np.testing.assert_allclose(E[:, 10], E[:, 38], rtol=1e-14)


@pytest.mark.parametrize("sub,n,K,seed", [(33, 32, 600, 0), (12, 8, 60, 1), (8, 6, 50, 7)])
def test_gradient_operator_bitwise_equal_to_oracle(sub, n, K, seed):
    """Finite strain (config 2): the 4-row displacement-gradient operator."""
    m = F.HyperRomModel(sub, n, K, seed)
    assert np.array_equal(m.G4, O.model_g4(sub, n, K, seed))


def test_finite_strain_paths_bitwise():
    H = F.make_paths(2, 0, 300, 30)
    assert H.shape == (300, 30, 4)
    assert np.array_equal(H, O.paths_fs(0, 300, 30))
    assert np.array_equal(F.make_paths(2, 0, 50, 30, p0=200), H[200:250])
