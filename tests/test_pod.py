"""POD basis from HF snapshots, CPU
side: the numpy POD oracle on the SPEC examples, the oracle's snapshot
recorder (rank of elastic snapshots, test_rve.cpp:258-294), the basis-driven
model build (host only) and the snapshot / basis containers."""
import numpy as np
import pytest

import pod_oracle as PO
import pyoracle as O
import paper_2306_02687_b200 as F
from paper_2306_02687_b200 import pod as P

DESK = [("j2", 1.0, 0.3, 0.01, 0.016), ("elastic", 10.0, 0.3)]


def _orth(rng, r, c):
    return np.linalg.qr(rng.standard_normal((c, r)))[0].T  # (r, c) orthonormal rows


def test_pod_all_in_elastic_span_has_no_extra_mode():
    rng = np.random.default_rng(0)
    Em = _orth(rng, 3, 200)
    X = rng.standard_normal((7, 3)) @ Em
    V, s, mx = PO.pod(X, 3, Em)
    assert mx == 3 and s.max() < 1e-12 * np.linalg.norm(X)
    with pytest.raises(ValueError):
        PO.pod(X, 4, Em)


def test_pod_single_orthogonal_column():
    rng = np.random.default_rng(1)
    Em = _orth(rng, 3, 120)
    v = rng.standard_normal(120)
    v -= Em.T @ (Em @ v)
    V, s, mx = PO.pod(v[None], 4, Em)
    u = v / np.linalg.norm(v)
    u *= np.sign(u[np.argmax(np.abs(u))])
    np.testing.assert_allclose(V[3], u, atol=1e-13)
    np.testing.assert_allclose(V[:3], Em, atol=1e-13)
    assert mx == 4


def test_pod_rank5_energy_fraction():
    rng = np.random.default_rng(2)
    X = rng.standard_normal((40, 5)) @ rng.standard_normal((5, 300))
    V, s, mx = PO.pod(X, 5)
    assert mx == 5
    assert abs(P.energy_fraction(s, 5) - 1.0) < 1e-12
    np.testing.assert_allclose(V @ V.T, np.eye(5), atol=1e-12)


def test_oracle_snapshots_elastic_range_rank3_and_counts():
    mesh = O.Mesh(0, 6)
    rng = np.random.default_rng(3)
    cols = []
    for _ in range(4):  # elastic range: |E| well below first yield (~0.01 / 1)
        end = rng.uniform(-1, 1, 3) * 2e-4
        r = mesh.hf_trajectory(DESK, np.stack([end * k / 5 for k in range(1, 6)]), snapshots=True)
        assert r["snapshots"].shape == (5, 2 * mesh.n_nodes)  # one column per increment
        cols.append(r["snapshots"])
    s = np.linalg.svd(np.concatenate(cols), compute_uv=False)
    assert (s[3:] < 1e-7 * s[0]).all() and s[2] > 1e-3 * s[0]
    # reconstructs in the elastic-mode span
    Em = PO.elastic_modes(mesh, DESK)
    assert len(Em) == 3
    np.testing.assert_allclose(Em @ Em.T, np.eye(3), atol=1e-12)
    X = np.concatenate(cols)
    resid = X - (X @ Em.T) @ Em
    assert np.linalg.norm(resid) <= 1e-8 * np.linalg.norm(X)


def test_oracle_elastic_modes_homogeneous_collapse():
    mesh = O.Mesh(geometry=1, subdivisions=4)
    assert len(PO.elastic_modes(mesh, [("elastic", 2.0, 0.25)])) == 0


def _free_index(xy):
    lo, hi = xy.min(axis=0), xy.max(axis=0)
    bnd = (np.abs(xy - lo) < 1e-12).any(axis=1) | (np.abs(xy - hi) < 1e-12).any(axis=1)
    fi = -np.ones(2 * len(xy), dtype=int)
    free = np.repeat(~bnd, 2)
    fi[free] = np.arange(free.sum())
    return fi


@pytest.mark.parametrize("sub,n,K", [(8, 6, 40), (12, 10, 0)])
def test_model_from_basis_equals_seeded_model(sub, n, K):
    """fe2_model_build_basis with the seeded Φ (expanded to all DOFs) rebuilds
    the seeded model bit for bit (host only)."""
    mesh = O.Mesh(0, sub)
    om = O.Model(sub, n, K, 5)
    fi = _free_index(mesh.xy)
    V = np.zeros((n, 2 * mesh.n_nodes))
    V[:, fi >= 0] = om.phi[fi[fi >= 0]].T
    V[:, fi < 0] = 1.0  # boundary rows are ignored under the linear BC
    a = F.HyperRomModel(sub, n, K, 5)
    b = F.HyperRomModel(sub, K=K, seed=5, basis=V)
    assert b.n == n and b.K == a.K
    np.testing.assert_array_equal(a.G, b.G)
    np.testing.assert_array_equal(a.G4, b.G4)
    np.testing.assert_array_equal(a.w, b.w)


def test_containers_round_trip(tmp_path):
    rng = np.random.default_rng(4)
    X = rng.standard_normal((6, 33))
    meta = [(t, k, (k + 1) / 3) for t in range(2) for k in range(3)]
    P.save_snapshots(tmp_path / "x.bin", X, meta)
    X2, meta2 = P.load_snapshots(tmp_path / "x.bin")
    np.testing.assert_array_equal(X, X2)
    assert meta2 == meta
    raw = (tmp_path / "x.bin").read_bytes()
    assert raw[:8] == b"FE2RMAT1" and len(raw) == 24 + 8 * X.size
    np.testing.assert_array_equal(np.frombuffer(raw[24:32], "<f8"), X[0, :1])  # column-major: column 0 first
    V = np.linalg.qr(rng.standard_normal((33, 4)))[0].T
    P.save_basis(tmp_path / "v.bin", V, [3.0, 2.0, 1.0], 3, source=X)
    V2, sv, ne, h = P.load_basis(tmp_path / "v.bin")
    np.testing.assert_array_equal(V, V2)
    assert ne == 3 and list(sv) == [3.0, 2.0, 1.0] and len(h) == 64
    (tmp_path / "bad.bin").write_bytes(b"nope")
    with pytest.raises(F.Fe2Error):
        P.load_matrix(tmp_path / "bad.bin")


def test_hf_requires_device():
    if F.device_count() > 0:
        pytest.skip("device present")
    with pytest.raises(F.Fe2Error):
        P.HfRve(8)
