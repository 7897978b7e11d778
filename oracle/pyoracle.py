"""ctypes wrapper of the CPU ORACLE (test infrastructure only).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this module — as the checker or as the
reference CPU arm, never as the product path.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "build", "liboracle.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_u8p = C.POINTER(C.c_uint8)


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        self.code = code
        super().__init__(f"oracle error {code}: {msg}")


class _Mat(C.Structure):
    _fields_ = [("kind", C.c_int), ("p", C.c_double * 6)]


class _Opts(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_iter", C.c_int), ("max_bisections", C.c_int)]


class _Out(C.Structure):
    _fields_ = [("sigma", _dp), ("C", _dp), ("iters", _ip), ("plastic_count", _ip), ("res_norm", _dp),
                ("status", _ip), ("bisections", _ip), ("plastic_flags", _u8p), ("alpha", _dp), ("state", _dp)]


def _load():
    if not os.path.exists(LIB_PATH):
        import subprocess
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    L = C.CDLL(LIB_PATH)
    L.orc_last_error.restype = C.c_char_p
    L.orc_rng_new.restype = C.c_void_p
    L.orc_rng_new.argtypes = [C.c_uint64]
    L.orc_rng_free.argtypes = [C.c_void_p]
    L.orc_rng_next_u64.restype = C.c_uint64
    L.orc_rng_next_u64.argtypes = [C.c_void_p]
    L.orc_rng_uniform.restype = C.c_double
    L.orc_rng_uniform.argtypes = [C.c_void_p]
    L.orc_rng_uniform_ab.restype = C.c_double
    L.orc_rng_uniform_ab.argtypes = [C.c_void_p, C.c_double, C.c_double]
    L.orc_rng_uniform_int.restype = C.c_int
    L.orc_rng_uniform_int.argtypes = [C.c_void_p, C.c_int]
    L.orc_rng_normal.restype = C.c_double
    L.orc_rng_normal.argtypes = [C.c_void_p]
    L.orc_update_material.argtypes = [C.POINTER(_Mat), _dp, _dp, _dp, _dp, _dp, _ip]
    L.orc_update4.argtypes = [C.POINTER(_Mat), _dp, _dp, _dp, _dp, _dp]
    L.orc_mesh_build.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_void_p)]
    L.orc_mesh_free.argtypes = [C.c_void_p]
    L.orc_mesh_counts.argtypes = [C.c_void_p, _ip, _ip, _dp]
    L.orc_mesh_arrays.argtypes = [C.c_void_p, _dp, _ip, _ip]
    L.orc_mesh_ip.argtypes = [C.c_void_p, C.c_int, _dp, _dp, _ip]
    L.orc_hf_trajectory.argtypes = [C.c_void_p, C.POINTER(_Mat), C.c_int, C.c_int, _dp, C.POINTER(_Opts), _dp, _dp,
                                    _ip, _dp, _dp, _dp]
    L.orc_model_build.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, C.POINTER(C.c_void_p)]
    L.orc_model_build_on_mesh.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_uint64, C.POINTER(C.c_void_p)]
    L.orc_model_free.argtypes = [C.c_void_p]
    L.orc_model_sizes.argtypes = [C.c_void_p, _ip, _ip, _ip, _dp]
    L.orc_model_arrays.argtypes = [C.c_void_p, _dp, _dp, _ip, _ip]
    L.orc_model_phi.argtypes = [C.c_void_p, _dp]
    L.orc_paths.argtypes = [C.c_int, C.c_uint64, C.c_int64, C.c_int64, C.c_int, _dp]
    L.orc_hrom_create.argtypes = [C.c_int, C.c_int, _dp, _dp, _ip, C.POINTER(_Mat), C.c_int, C.c_double,
                                  C.POINTER(C.c_void_p)]
    L.orc_hrom_free.argtypes = [C.c_void_p]
    L.orc_hrom_run.argtypes = [C.c_void_p, C.c_int64, C.c_int, _dp, C.POINTER(_Opts), C.c_int, C.POINTER(_Out)]
    L.orc_hrom_assemble.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _ip, _dp]
    return L


lib = _load()


def _check(rc):
    if rc != 0:
        raise OracleError(rc, lib.orc_last_error().decode())


def _d(a):
    return None if a is None else a.ctypes.data_as(_dp)


def _i(a):
    return None if a is None else a.ctypes.data_as(_ip)


def mat_struct(m):
    """m: ('elastic', E, nu) | ('j2', E, nu, sy0, h) | ('powerlaw', E, nu, sy0, N)
    | ('creep', E, nu, A, n, m, dt), or an object with the product's fields."""
    def mk(kind, *p):
        return _Mat(kind, (C.c_double * 6)(*(list(p) + [0.0] * (6 - len(p)))))
    if hasattr(m, "hardening"):
        return mk(1, m.E, m.nu, m.sigma_y0, m.hardening)
    if hasattr(m, "N"):
        return mk(2, m.E, m.nu, m.sigma_y0, m.N)
    if hasattr(m, "A"):
        return mk(3, m.E, m.nu, m.A, m.n, m.m, m.dt)
    if hasattr(m, "E"):
        return mk(0, m.E, m.nu)
    kinds = {"elastic": 0, "j2": 1, "powerlaw": 2, "creep": 3}
    return mk(kinds[m[0]], *m[1:])


class Rng:
    def __init__(self, seed):
        self._h = lib.orc_rng_new(seed)

    def __del__(self):
        if getattr(self, "_h", None):
            lib.orc_rng_free(self._h)

    def next_u64(self):
        return lib.orc_rng_next_u64(self._h)

    def uniform(self, a=None, b=None):
        if a is None:
            return lib.orc_rng_uniform(self._h)
        return lib.orc_rng_uniform_ab(self._h, a, b)

    def uniform_int(self, n):
        return lib.orc_rng_uniform_int(self._h, n)

    def normal(self):
        return lib.orc_rng_normal(self._h)


def update_material(mat, state, eps):
    """Returns sigma(3), C(3,3), state_out(6), plastic(bool)."""
    m = mat_struct(mat)
    st = np.zeros(6) if state is None else np.ascontiguousarray(state, dtype=np.float64)
    e = np.ascontiguousarray(eps, dtype=np.float64)
    s, Cm, so, pl = np.empty(3), np.empty((3, 3)), np.empty(6), C.c_int()
    _check(lib.orc_update_material(C.byref(m), _d(st), _d(e), _d(s), _d(Cm), _d(so), C.byref(pl)))
    return s, Cm, so, bool(pl.value)


def update4(mat, state, eps4):
    m = mat_struct(mat)
    st = np.zeros(6) if state is None else np.ascontiguousarray(state, dtype=np.float64)
    e = np.ascontiguousarray(eps4, dtype=np.float64)
    s, D, so = np.empty(4), np.empty((4, 4)), np.empty(6)
    _check(lib.orc_update4(C.byref(m), _d(st), _d(e), _d(s), _d(D), _d(so)))
    return s, D, so


class Mesh:
    def __init__(self, geometry=0, subdivisions=8):
        h = C.c_void_p()
        _check(lib.orc_mesh_build(geometry, subdivisions, C.byref(h)))
        self._h = h
        nn, ne, area = C.c_int(), C.c_int(), C.c_double()
        lib.orc_mesh_counts(h, C.byref(nn), C.byref(ne), C.byref(area))
        self.n_nodes, self.n_elements, self.area = nn.value, ne.value, area.value
        self.xy = np.empty((self.n_nodes, 2))
        self.conn = np.empty((self.n_elements, 6), dtype=np.int32)
        self.mat = np.empty(self.n_elements, dtype=np.int32)
        lib.orc_mesh_arrays(h, _d(self.xy), _i(self.conn), _i(self.mat))

    def __del__(self):
        if getattr(self, "_h", None):
            lib.orc_mesh_free(self._h)

    def ip(self, i):
        B, w, e = np.empty((3, 12)), C.c_double(), C.c_int()
        _check(lib.orc_mesh_ip(self._h, i, _d(B), C.byref(w), C.byref(e)))
        return B, w.value, e.value

    def hf_trajectory(self, materials, E_path, tol=1e-8, max_iter=30, max_bisections=4, snapshots=False):
        E_path = np.ascontiguousarray(E_path, dtype=np.float64).reshape(-1, 3)
        k = E_path.shape[0]
        mats = (_Mat * len(materials))(*[mat_struct(m) for m in materials])
        o = _Opts(tol, max_iter, max_bisections)
        sig, Cm, it = np.empty((k, 3)), np.empty((k, 3, 3)), np.empty(k, dtype=np.int32)
        uf, rl = np.empty(k), np.empty(k)
        X = np.empty((k, 2 * self.n_nodes)) if snapshots else None
        _check(lib.orc_hf_trajectory(self._h, mats, len(materials), k, _d(E_path), C.byref(o), _d(sig), _d(Cm),
                                     _i(it), _d(uf), _d(rl), _d(X) if snapshots else None))
        out = dict(sigma=sig, C=Cm, iterations=it, u_fluct_inf=uf, res_last=rl)
        if snapshots:
            out["snapshots"] = X
        return out


class Model:
    def __init__(self, subdivisions=33, n=12, K=200, seed=0, mesh: Mesh | None = None):
        h = C.c_void_p()
        if mesh is None:
            _check(lib.orc_model_build(subdivisions, n, K, seed, C.byref(h)))
        else:
            _check(lib.orc_model_build_on_mesh(mesh._h, n, K, seed, C.byref(h)))
        try:
            n_, K_, nf, vol = C.c_int(), C.c_int(), C.c_int(), C.c_double()
            lib.orc_model_sizes(h, C.byref(n_), C.byref(K_), C.byref(nf), C.byref(vol))
            self.n, self.K, self.n_free, self.volume = n_.value, K_.value, nf.value, vol.value
            self.G = np.empty((self.K, 3, self.n))
            self.w = np.empty(self.K)
            self.ip = np.empty(self.K, dtype=np.int32)
            self.mat = np.empty(self.K, dtype=np.int32)
            lib.orc_model_arrays(h, _d(self.G), _d(self.w), _i(self.ip), _i(self.mat))
            self.phi = np.empty((self.n_free, self.n))
            lib.orc_model_phi(h, _d(self.phi))
        finally:
            lib.orc_model_free(h)


def paths(kind, seed, P, n_incr, p0=0):
    E = np.empty((P, n_incr, 3))
    _check(lib.orc_paths(kind, seed, p0, P, n_incr, _d(E)))
    return E


class Hrom:
    """The oracle's hyper-ROM online path on given model arrays."""

    def __init__(self, G, w, mat_id, materials, volume):
        G = np.ascontiguousarray(G, dtype=np.float64)
        self.K, _, self.n = G.shape
        w = np.ascontiguousarray(w, dtype=np.float64)
        mid = np.ascontiguousarray(mat_id, dtype=np.int32)
        mats = (_Mat * len(materials))(*[mat_struct(m) for m in materials])
        h = C.c_void_p()
        _check(lib.orc_hrom_create(self.n, self.K, _d(G), _d(w), _i(mid), mats, len(materials), float(volume),
                                   C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            lib.orc_hrom_free(self._h)

    def run(self, E, tol=1e-8, max_iter=30, max_bisections=4, threads=1, flags=False, final_state=False):
        E = np.ascontiguousarray(E, dtype=np.float64)
        P, k, _ = E.shape
        res = dict(sigma=np.empty((P, k, 3)), C=np.empty((P, k, 3, 3)), iters=np.empty((P, k), dtype=np.int32),
                   plastic_count=np.empty((P, k), dtype=np.int32), res_norm=np.empty((P, k)),
                   status=np.empty((P, k), dtype=np.int32), bisections=np.empty((P, k), dtype=np.int32))
        if flags:
            res["plastic_flags"] = np.empty((P, k, self.K), dtype=np.uint8)
        if final_state:
            res["alpha"] = np.empty((P, self.n))
            res["state"] = np.empty((P, self.K, 6))
        o = _Out(_d(res["sigma"]), _d(res["C"]), _i(res["iters"]), _i(res["plastic_count"]), _d(res["res_norm"]),
                 _i(res["status"]), _i(res["bisections"]),
                 res["plastic_flags"].ctypes.data_as(_u8p) if flags else None,
                 _d(res.get("alpha")), _d(res.get("state")))
        opts = _Opts(tol, max_iter, max_bisections)
        _check(lib.orc_hrom_run(self._h, P, k, _d(E), C.byref(opts), threads, C.byref(o)))
        return res

    def assemble(self, alpha, E, state=None):
        n = self.n
        alpha = np.ascontiguousarray(alpha, dtype=np.float64)
        E = np.ascontiguousarray(E, dtype=np.float64)
        st = None if state is None else np.ascontiguousarray(state, dtype=np.float64)
        r, Kaa, KaE, CEE, S, pc = np.empty(n), np.empty((n, n)), np.empty((n, 3)), np.empty((3, 3)), np.empty(3), C.c_int()
        so = np.empty((self.K, 6))
        _check(lib.orc_hrom_assemble(self._h, _d(alpha), _d(E), _d(st), _d(r), _d(Kaa), _d(KaE), _d(CEE), _d(S),
                                     C.byref(pc), _d(so)))
        return dict(r=r, Kaa=Kaa, KaE=KaE, C_EE=CEE, S_raw=S, plastic_count=pc.value, state=so)


# ---- finite strain, Biot stress (config 2; parity unpinned) ----------------
lib.orc_update_biot.argtypes = [C.POINTER(_Mat), _dp, _dp, _dp, _dp, _dp, _ip]
lib.orc_model_g4.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, _dp]
lib.orc_paths_fs.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.c_int, _dp]
lib.orc_hrom_fs_create.argtypes = [C.c_int, C.c_int, _dp, _dp, _ip, C.POINTER(_Mat), C.c_int, C.c_double,
                                   C.POINTER(C.c_void_p)]
lib.orc_hrom_fs_free.argtypes = [C.c_void_p]
lib.orc_hrom_fs_run.argtypes = [C.c_void_p, C.c_int64, C.c_int, _dp, C.POINTER(_Opts), C.c_int, C.POINTER(_Out)]
lib.orc_hrom_fs_assemble.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _ip]


def update_biot(mat, state, F4):
    """Returns P(4), A(4,4), state_out(6), plastic."""
    m = mat_struct(mat)
    st = np.zeros(6) if state is None else np.ascontiguousarray(state, dtype=np.float64)
    F = np.ascontiguousarray(F4, dtype=np.float64)
    P, A, so, pl = np.empty(4), np.empty((4, 4)), np.empty(6), C.c_int()
    _check(lib.orc_update_biot(C.byref(m), _d(st), _d(F), _d(P), _d(A), _d(so), C.byref(pl)))
    return P, A, so, bool(pl.value)


def model_g4(subdivisions, n, K, seed):
    G4 = np.empty((K, 4, n))
    _check(lib.orc_model_g4(subdivisions, n, K, seed, _d(G4)))
    return G4


def paths_fs(seed, P, n_incr, p0=0):
    H = np.empty((P, n_incr, 4))
    _check(lib.orc_paths_fs(seed, p0, P, n_incr, _d(H)))
    return H


class HromFs:
    """Oracle of the finite-strain (Biot) hyper-ROM path."""

    def __init__(self, G4, w, mat_id, materials, volume):
        G4 = np.ascontiguousarray(G4, dtype=np.float64)
        self.K, _, self.n = G4.shape
        w = np.ascontiguousarray(w, dtype=np.float64)
        mid = np.ascontiguousarray(mat_id, dtype=np.int32)
        mats = (_Mat * len(materials))(*[mat_struct(m) for m in materials])
        h = C.c_void_p()
        _check(lib.orc_hrom_fs_create(self.n, self.K, _d(G4), _d(w), _i(mid), mats, len(materials), float(volume),
                                      C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            lib.orc_hrom_fs_free(self._h)

    def run(self, H, tol=1e-8, max_iter=30, max_bisections=4, threads=1, flags=False, final_state=False):
        H = np.ascontiguousarray(H, dtype=np.float64)
        P, k, _ = H.shape
        res = dict(P=np.empty((P, k, 4)), A=np.empty((P, k, 4, 4)), iters=np.empty((P, k), dtype=np.int32),
                   plastic_count=np.empty((P, k), dtype=np.int32), res_norm=np.empty((P, k)),
                   status=np.empty((P, k), dtype=np.int32), bisections=np.empty((P, k), dtype=np.int32))
        if flags:
            res["plastic_flags"] = np.zeros((P, k, self.K), dtype=np.uint8)
        if final_state:
            res["alpha"] = np.empty((P, self.n))
            res["state"] = np.empty((P, self.K, 6))
        o = _Out(_d(res["P"]), _d(res["A"]), _i(res["iters"]), _i(res["plastic_count"]), _d(res["res_norm"]),
                 _i(res["status"]), _i(res["bisections"]),
                 res["plastic_flags"].ctypes.data_as(_u8p) if flags else None,
                 _d(res.get("alpha")), _d(res.get("state")))
        opts = _Opts(tol, max_iter, max_bisections)
        _check(lib.orc_hrom_fs_run(self._h, P, k, _d(H), C.byref(opts), threads, C.byref(o)))
        return res

    def assemble(self, alpha, H, state=None):
        n = self.n
        alpha = np.ascontiguousarray(alpha, dtype=np.float64)
        H = np.ascontiguousarray(H, dtype=np.float64)
        st = None if state is None else np.ascontiguousarray(state, dtype=np.float64)
        r, Kaa, KaF, KFa = np.empty(n), np.empty((n, n)), np.empty((n, 4)), np.empty((4, n))
        CFF, Praw, pc = np.empty((4, 4)), np.empty(4), C.c_int()
        _check(lib.orc_hrom_fs_assemble(self._h, _d(alpha), _d(H), _d(st), _d(r), _d(Kaa), _d(KaF), _d(KFa), _d(CFF),
                                        _d(Praw), C.byref(pc)))
        return dict(r=r, Kaa=Kaa, KaF=KaF, KFa=KFa, C_FF=CFF, P_raw=Praw, plastic_count=pc.value)
