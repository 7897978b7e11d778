"""CPU ORACLE of the POD basis construction (test infrastructure only).

Restates, in numpy, rom.build_elastic_modes and rom.pod on
top of the oracle's HF trajectory (orc_hf_trajectory, the run_trajectory +
SnapshotRecorder restatement, rve.hpp:397-494):
  elastic modes  = x_u of one elastic step to each unit macro strain,
                   Gram-Schmidt (twice), dropped below 1e-10 |E.x|;
  pod            = [elastic | leading left singular vectors of X deflated
                   against the elastic span], re-orthonormalised; a POD mode's
                   largest-magnitude entry is positive; rank = #s > 1e-10 |X|_F.
The reference leaves the SVD algorithm open (Eigen in the reference build);
numpy's LAPACK SVD is the checker here.
"""
from __future__ import annotations

import numpy as np

import pyoracle as O


def orthonormalize(A, drop):
    """Modified Gram-Schmidt, twice per column; columns of A are rows of the array."""
    out = []
    for j, v in enumerate(np.array(A, dtype=np.float64)):
        for _ in range(2):
            for q in out:
                v = v - (q @ v) * q
        nrm = np.linalg.norm(v)
        if nrm > drop[j]:
            out.append(v / nrm)
    return np.array(out).reshape(len(out), np.shape(A)[1])


def affine(mesh: O.Mesh, E):
    u = np.zeros(2 * mesh.n_nodes)
    u[0::2] = E[0] * mesh.xy[:, 0] + 0.5 * E[2] * mesh.xy[:, 1]
    u[1::2] = 0.5 * E[2] * mesh.xy[:, 0] + E[1] * mesh.xy[:, 1]
    return u


def elastic_part(m):
    return ("elastic", m[1], m[2]) if m[0] == "j2" else m


def elastic_modes(mesh: O.Mesh, materials):
    mats = [elastic_part(m) for m in materials]
    cols, drop = [], []
    for j in range(3):
        E = np.zeros(3)
        E[j] = 1.0
        r = mesh.hf_trajectory(mats, E[None], tol=1e-10, max_iter=10, max_bisections=0, snapshots=True)
        cols.append(r["snapshots"][0])
        drop.append(1e-10 * np.linalg.norm(affine(mesh, E)))
    return orthonormalize(cols, drop)


def pod(X, n_target, elastic=None):
    """X (n_cols, n_rows), elastic (n_e, n_rows) -> V (n_target, n_rows), s, max modes."""
    X = np.asarray(X, dtype=np.float64)
    Em = np.zeros((0, X.shape[1])) if elastic is None else orthonormalize(elastic, [1e-10] * len(elastic))
    ne = len(Em)
    D = X.copy()
    for _ in range(2):
        D = D - (D @ Em.T) @ Em
    U, s, _ = np.linalg.svd(D.T, full_matrices=False)
    rank = int(np.sum(s > 1e-10 * np.linalg.norm(X)))
    k = n_target - ne
    if k > rank:
        raise ValueError(f"rank: at most {ne + rank} modes usable")
    V = orthonormalize(np.concatenate([Em, U[:, :k].T]), [1e-8] * n_target)
    for j in range(ne, n_target):
        i = int(np.argmax(np.abs(V[j])))
        if V[j, i] < 0:
            V[j] = -V[j]
    sv = np.zeros(X.shape[0])
    sv[:len(s)] = s
    return V, sv, ne + rank
