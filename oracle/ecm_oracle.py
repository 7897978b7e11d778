"""CPU ORACLE of the ECM point selection (test infrastructure only):
numpy restatement of fe2_ecm_select (SPEC.md:333-369 hyper.ecm_select;
greedy max-correlation selection, least-squares re-fit, removal of
non-positive weights, constant column for volume exactness)."""
import numpy as np


def ecm_select(U, w_full, m_target, tol):
    U = np.asarray(U, dtype=np.float64)
    m, k = U.shape
    cscale = np.abs(U).max() if U.size and np.abs(U).max() > 0 else 1.0 / np.sqrt(m)
    Ue = np.concatenate([U, np.full((m, 1), cscale)], axis=1)
    b = Ue.T @ w_full
    bn = np.linalg.norm(b)
    rn = np.linalg.norm(Ue, axis=1)
    Z, w, r = [], np.zeros(0), b.copy()
    alive = rn > 0
    while len(Z) < min(m_target, k + 1) and np.linalg.norm(r) / bn > tol:
        c = np.where(alive, Ue @ r / np.where(rn > 0, rn, 1.0), -np.inf)
        c[Z] = -np.inf
        q = int(np.argmax(c))
        if not c[q] > 0:
            break
        Z.append(q)
        while Z:
            A = Ue[Z].T
            w = np.linalg.lstsq(A, b, rcond=None)[0]
            keep = [z for z, x in zip(Z, w) if x > 0]
            if len(keep) == len(Z):
                break
            Z = keep
        r = b - Ue[Z].T @ w
    order = np.argsort(Z)
    return np.array(Z)[order], w[order], np.linalg.norm(r) / bn
