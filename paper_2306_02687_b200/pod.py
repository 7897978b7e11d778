"""Offline POD basis from high-fidelity RVE snapshots (
SPEC.md:256-316 rom.build_elastic_modes / rom.pod): the full-field micro
problem solved on the device (fe2_hf_*: element kernel + deterministic band
assembly + band Cholesky on one CTA per system, many trajectories at once),
x_u snapshot columns per converged increment
(run_trajectory + SnapshotRecorder, rve.hpp:397-494), elastic modes prepended,
SVD of the deflated snapshots (fe2_pod_basis), and the hyper-ROM model built
on that basis (fe2_model_build_basis). Plus the binary container + text
manifest persistence of snapshot and basis matrices.
Offline tooling around the online engine; no CPU fallback."""
from __future__ import annotations

import ctypes as C
import hashlib
import struct

import numpy as np

from .hrom import ElasticParams, Fe2Error, HyperRomModel, J2LinearParams, NewtonOptions, _check, _d, _i, lib

DESK = (J2LinearParams(1.0, 0.3, 0.01, 0.016), ElasticParams(10.0, 0.3))


class HfRve:
    """High-fidelity RVE on one device (micro_newton + homogenize +
    run_trajectory, rve.hpp:285-494, linear BC). RVE = default_cell
    (subdivisions) or a mesh file; materials indexed by element material id."""

    def __init__(self, subdivisions=33, materials=DESK, mesh_file: str | None = None, device=0):
        from .hrom import _Material
        mats = (_Material * len(materials))(*[m._c() for m in materials])
        h = C.c_void_p()
        path = None if mesh_file is None else str(mesh_file).encode()
        _check(lib.fe2_hf_create(device, subdivisions, path, mats, len(materials), C.byref(h)))
        self._h = h
        nd, nf, nip, vol = C.c_int(), C.c_int(), C.c_int(), C.c_double()
        _check(lib.fe2_hf_sizes(h, C.byref(nd), C.byref(nf), C.byref(nip), C.byref(vol)))
        self.n_dofs, self.n_free, self.n_ips, self.volume = nd.value, nf.value, nip.value, vol.value

    def __del__(self):
        if getattr(self, "_h", None):
            lib.fe2_hf_destroy(self._h)
            self._h = None

    def trajectory(self, E_path, opts: NewtonOptions | None = None, snapshots=True):
        """Strain path E_path (k, 3) from the virgin state. Returns sigma (k,3),
        C (k,3,3), iterations (k,), u_fluct_inf, res_last and, with
        snapshots, the x_u columns (k, n_dofs) = u - E.x per step."""
        E_path = np.ascontiguousarray(E_path, dtype=np.float64).reshape(-1, 3)
        k = E_path.shape[0]
        o = (opts or NewtonOptions())._c()
        sig, Cm, it = np.empty((k, 3)), np.empty((k, 3, 3)), np.empty(k, dtype=np.int32)
        uf, rl = np.empty(k), np.empty(k)
        X = np.empty((k, self.n_dofs)) if snapshots else None
        _check(lib.fe2_hf_trajectory(self._h, k, _d(E_path), C.byref(o), _d(sig), _d(Cm), _i(it), _d(uf), _d(rl),
                                     _d(X)))
        out = dict(sigma=sig, C=Cm, iterations=it, u_fluct_inf=uf, res_last=rl)
        if snapshots:
            out["snapshots"] = X
        return out

    def trajectories(self, E_paths, opts: NewtonOptions | None = None, snapshots=True):
        """A batch of independent strain paths E_paths (T, k, 3), each from the
        virgin state, solved concurrently (fe2_hf_trajectories). Returns the
        trajectory() fields stacked over T plus status (T,) (0 or 1 + ErrorCode)."""
        E_paths = np.ascontiguousarray(E_paths, dtype=np.float64)
        T, k = E_paths.shape[:2]
        o = (opts or NewtonOptions())._c()
        sig, Cm, it = np.empty((T, k, 3)), np.empty((T, k, 3, 3)), np.empty((T, k), dtype=np.int32)
        uf, rl, st = np.empty((T, k)), np.empty((T, k)), np.empty(T, dtype=np.int32)
        X = np.empty((T, k, self.n_dofs)) if snapshots else None
        _check(lib.fe2_hf_trajectories(self._h, T, k, _d(E_paths), C.byref(o), _d(sig), _d(Cm), _i(it), _d(uf),
                                       _d(rl), _d(X), _i(st)))
        out = dict(sigma=sig, C=Cm, iterations=it, u_fluct_inf=uf, res_last=rl, status=st)
        if snapshots:
            out["snapshots"] = X
        return out

    @property
    def half_bandwidth(self):
        """Half bandwidth of the free stiffness in the device's band (RCM) ordering."""
        b = C.c_int()
        _check(lib.fe2_hf_band(self._h, C.byref(b)))
        return b.value

    # ---- HF engine of an FE² run: P macro points with their own states
    def alloc_points(self, P):
        """P macro points in the virgin state (fe2_hf_alloc_points)."""
        _check(lib.fe2_hf_alloc_points(self._h, P))
        self.P = P

    def solve_increment(self, E, opts: NewtonOptions | None = None):
        """One path step for every point from its committed state: E (P,3) ->
        sigma (P,3), C (P,3,3), iters, status (0 or 1 + ErrorCode)."""
        E = np.ascontiguousarray(E, dtype=np.float64).reshape(self.P, 3)
        o = (opts or NewtonOptions())._c()
        sig, Cm = np.empty((self.P, 3)), np.empty((self.P, 3, 3))
        it, st = np.empty(self.P, dtype=np.int32), np.empty(self.P, dtype=np.int32)
        _check(lib.fe2_hf_solve_increment(self._h, _d(E), C.byref(o), _d(sig), _d(Cm), _i(it), _i(st)))
        return dict(sigma=sig, C=Cm, iters=it, status=st)

    def mono_begin(self):
        """HF_monolithic: start a step from the committed state."""
        _check(lib.fe2_hf_mono_begin(self._h))

    def mono_iterate(self, E):
        """One condensed full-field Newton iteration of every point at macro strains
        E (P,3): sigma (P,3), C (P,3,3), rel_res, status (fe2_hf_mono_iterate)."""
        E = np.ascontiguousarray(E, dtype=np.float64).reshape(self.P, 3)
        sig, Cm, rr = np.empty((self.P, 3)), np.empty((self.P, 3, 3)), np.empty(self.P)
        st = np.empty(self.P, dtype=np.int32)
        _check(lib.fe2_hf_mono_iterate(self._h, _d(E), _d(sig), _d(Cm), _d(rr), _i(st)))
        return dict(sigma=sig, C=Cm, rel_res=rr, status=st)

    def mono_commit(self):
        _check(lib.fe2_hf_mono_commit(self._h))

    def snapshot(self):
        _check(lib.fe2_hf_snapshot(self._h))

    def restore(self):
        _check(lib.fe2_hf_restore(self._h))

    def elastic_modes(self):
        """build_elastic_modes: (count, n_dofs) orthonormal
        fluctuation responses to unit macro strains; 0 rows for a homogeneous RVE."""
        M = np.empty((3, self.n_dofs))
        cnt = C.c_int()
        _check(lib.fe2_hf_elastic_modes(self._h, _d(M), C.byref(cnt)))
        return M[:cnt.value].copy()


def pod_basis(X, n_target, elastic=None, device=0):
    """pod. X (n_cols, n_rows): snapshot columns as rows;
    elastic (n_e, n_rows). Returns V (n_target, n_rows) orthonormal = [elastic |
    POD modes], the deflated singular values (n_cols,), and the largest usable
    mode count. Asking for more than that raises Fe2Error (kind "rank")."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    n_cols, n_rows = X.shape
    Em = None if elastic is None or len(elastic) == 0 else np.ascontiguousarray(elastic, dtype=np.float64)
    ne = 0 if Em is None else Em.shape[0]
    V = np.empty((n_target, n_rows))
    sv = np.empty(n_cols)
    mx = C.c_int(-1)
    _check(lib.fe2_pod_basis(device, _d(X), n_rows, n_cols, _d(Em), ne, n_target, _d(V), _d(sv), C.byref(mx)))
    return V, sv, mx.value


def max_usable_modes(X, elastic=None, device=0):
    """n_elastic + rank of the deflated snapshots (the pod rank error's bound)."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    Em = None if elastic is None or len(elastic) == 0 else np.ascontiguousarray(elastic, dtype=np.float64)
    ne = 0 if Em is None else Em.shape[0]
    V, sv, mx = np.empty((max(1, ne), X.shape[1])), np.empty(X.shape[0]), C.c_int(-1)
    rc = lib.fe2_pod_basis(device, _d(X), X.shape[1], X.shape[0], _d(Em), ne, max(1, ne), _d(V), _d(sv), C.byref(mx))
    if rc not in (0, 7):  # 7 = 1 + ErrorCode::rank
        _check(rc)
    return mx.value


def energy_fraction(singular_values, k):
    """Σ_{i<k} s_i² / Σ s_i² of the deflated snapshots."""
    s2 = np.asarray(singular_values, dtype=np.float64) ** 2
    tot = s2.sum()
    return 1.0 if tot == 0.0 else float(s2[:k].sum() / tot)


def monotonic_path(end, n_steps=20):
    """make_monotonic_path (rve.hpp:426-435): step i = (i / n) end."""
    end = np.asarray(end, dtype=np.float64)
    return np.stack([end * (k / n_steps) for k in range(1, n_steps + 1)])


def collect_snapshots(rve: HfRve, endpoints, n_steps=20, opts: NewtonOptions | None = None):
    """Monotonic training trajectories to each endpoint:
    x_u columns (n_traj * n_steps, n_dofs) and their manifest rows
    (trajectory, increment, load factor)."""
    ends = np.atleast_2d(endpoints)
    r = rve.trajectories(np.stack([monotonic_path(e, n_steps) for e in ends]), opts)  # concurrently
    bad = np.flatnonzero(r["status"])
    if bad.size:
        raise Fe2Error(int(r["status"][bad[0]]), lib.fe2_last_error().decode())
    meta = [(t, k, (k + 1) / n_steps) for t in range(len(ends)) for k in range(n_steps)]
    return r["snapshots"].reshape(-1, rve.n_dofs), meta


def train_model(rve: HfRve, endpoints, n_modes, K=0, seed=0, n_steps=20, subdivisions=33, mesh_file=None, device=0):
    """Training trajectories -> elastic modes + POD -> hyper-ROM model on the
    physical basis (K = 0: full rule; else seeded cubature). Returns (model, V, sv)."""
    X, _ = collect_snapshots(rve, endpoints, n_steps)
    V, sv, _ = pod_basis(X, n_modes, rve.elastic_modes(), device)
    return HyperRomModel(subdivisions, K=K, seed=seed, mesh_file=mesh_file, basis=V), V, sv


# ---- persistence: binary container + text manifest ----
_MAGIC = b"FE2RMAT1"


def save_matrix(path, cols):
    """Column-major container: magic, int64 rows, int64 cols, doubles.
    cols (n_cols, n_rows) holds one column per row of the array."""
    cols = np.ascontiguousarray(cols, dtype="<f8")
    with open(path, "wb") as f:
        f.write(_MAGIC + struct.pack("<qq", cols.shape[1], cols.shape[0]))
        f.write(cols.tobytes())


def load_matrix(path):
    with open(path, "rb") as f:
        head = f.read(24)
        if len(head) != 24 or head[:8] != _MAGIC:
            raise Fe2Error(9, f"not a fe2rom matrix container: {path}")
        rows, cols = struct.unpack("<qq", head[8:])
        data = np.frombuffer(f.read(), dtype="<f8")
    if data.size != rows * cols:
        raise Fe2Error(9, f"truncated matrix container: {path}")
    return data.reshape(cols, rows).astype(np.float64)


def save_snapshots(path, X, meta):
    save_matrix(path, X)
    with open(str(path) + ".manifest", "w") as f:
        f.write("# column trajectory increment load_factor\n")
        for c, (t, k, lf) in enumerate(meta):
            f.write(f"{c} {t} {k} {lf:.17g}\n")


def load_snapshots(path):
    X = load_matrix(path)
    meta = []
    with open(str(path) + ".manifest") as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            _, t, k, lf = line.split()
            meta.append((int(t), int(k), float(lf)))
    if len(meta) != X.shape[0]:
        raise Fe2Error(9, "snapshot manifest does not match the container")
    return X, meta


def save_basis(path, V, singular_values, n_elastic, source=None):
    """Basis container + manifest (ñ, elastic count, singular values, source
    snapshot hash — SPEC.md:311)."""
    save_matrix(path, V)
    src = "none" if source is None else hashlib.sha256(np.ascontiguousarray(source, dtype="<f8").tobytes()).hexdigest()
    with open(str(path) + ".manifest", "w") as f:
        f.write(f"modes {V.shape[0]}\nelastic {n_elastic}\nsource_sha256 {src}\n")
        f.write("singular_values " + " ".join(f"{s:.17g}" for s in singular_values) + "\n")


def load_basis(path):
    V = load_matrix(path)
    info = {}
    with open(str(path) + ".manifest") as f:
        for line in f:
            key, _, rest = line.strip().partition(" ")
            info[key] = rest
    if int(info["modes"]) != V.shape[0]:
        raise Fe2Error(9, "basis manifest does not match the container")
    sv = np.array([float(x) for x in info.get("singular_values", "").split()])
    return V, sv, int(info["elastic"]), info["source_sha256"]
