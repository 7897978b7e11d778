"""ctypes mirror of the reference interface over the native C ABI.

Reference names kept (paths relative to /root/reference/proj/include/fe2rom/):
  ElasticParams / J2LinearParams          materials.hpp:37-49
  update_material (batched)               materials.hpp:317-325
  MicroOptions {tol, max_iter} + max_bisections   rve.hpp:195-200, :439-443
  run_trajectory step per macro point     rve.hpp:448-494 (reduced: SPEC.md:289-297)
Errors: Fe2Error carries the reference ErrorCode name (common.hpp:26-37).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FE2_LIB") or os.path.join(_HERE, "lib", "libfe2rom_gpu.so")

ERROR_CODES = ["config", "geometry", "mesh", "material", "solver", "numeric", "rank", "bc", "io", "provenance"]

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_u8p = C.POINTER(C.c_uint8)


class Fe2Error(RuntimeError):
    def __init__(self, code: int, msg: str):
        self.code = code
        self.kind = ERROR_CODES[code - 1] if 1 <= code <= len(ERROR_CODES) else f"code{code}"
        super().__init__(f"[{self.kind}] {msg}")


class _Material(C.Structure):
    _fields_ = [("kind", C.c_int), ("p", C.c_double * 6)]


class _Opts(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_iter", C.c_int), ("max_bisections", C.c_int)]


class _Stats(C.Structure):
    _fields_ = [
        ("points", C.c_int64),
        ("n", C.c_int),
        ("K", C.c_int),
        ("K_j2", C.c_int),
        ("kernel_launches", C.c_int64),
        ("increments", C.c_int64),
        ("assemblies", C.c_int64),
        ("commits", C.c_int64),
        ("plastic_evals", C.c_int64),
        ("kernel_ms", C.c_double),
        ("timed_launches", C.c_int64),
        ("timed_assemblies", C.c_int64),
        ("timed_commits", C.c_int64),
        ("timed_plastic_evals", C.c_int64),
        ("timed_commit_plastic", C.c_int64),
    ]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"native library missing: {LIB_PATH} — run __graft_entry__.build() "
            "(there is no CPU fallback for the hyper-ROM engine)"
        )
    L = C.CDLL(LIB_PATH)
    L.fe2_last_error.restype = C.c_char_p
    L.fe2_version.restype = C.c_char_p
    L.fe2_device_count.restype = C.c_int
    L.fe2_material_update_batch.argtypes = [C.c_int, C.POINTER(_Material), C.c_int64, _dp, _dp, _dp, _dp, _dp, _u8p]
    L.fe2_material_update_soa_device.argtypes = [C.c_int, C.POINTER(_Material), C.c_int64] + [C.c_void_p] * 7
    L.fe2_hrom_create.argtypes = [C.c_int, C.c_int, C.c_int, _dp, _dp, _ip, C.POINTER(_Material), C.c_int, C.c_double,
                                  C.POINTER(C.c_void_p)]
    L.fe2_hrom_create_fs.argtypes = L.fe2_hrom_create.argtypes
    L.fe2_hrom_kinematics.argtypes = [C.c_void_p, _ip]
    L.fe2_hrom_fs_assemble_point.argtypes = [C.c_void_p, C.c_int64, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp]
    L.fe2_model_g4.argtypes = [C.c_void_p, _dp]
    L.fe2_hrom_destroy.argtypes = [C.c_void_p]
    L.fe2_hrom_destroy.restype = None
    L.fe2_hrom_alloc_points.argtypes = [C.c_void_p, C.c_int64, C.c_int]
    L.fe2_hrom_solve_increment.argtypes = [C.c_void_p, _dp, C.POINTER(_Opts), _dp, _dp, _ip, _ip, _dp, _ip]
    L.fe2_hrom_solve_increment_async.argtypes = [C.c_void_p, _dp, C.POINTER(_Opts), _dp, _dp, _ip, _ip, _dp, _ip]
    L.fe2_hrom_wait.argtypes = [C.c_void_p]
    L.fe2_hrom_solve_increment_device.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(_Opts), C.c_void_p, C.c_void_p,
                                                  C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    L.fe2_hrom_read_state.argtypes = [C.c_void_p, _dp, _dp, _u8p]
    L.fe2_hrom_assemble_point.argtypes = [C.c_void_p, C.c_int64, _dp, _dp, _dp, _dp, _dp, _dp, _dp]
    L.fe2_hrom_stats.argtypes = [C.c_void_p, C.POINTER(_Stats)]
    L.fe2_hrom_set_timing.argtypes = [C.c_void_p, C.c_int]
    L.fe2_hrom_reset_stats.argtypes = [C.c_void_p]
    L.fe2_hrom_set_stream.argtypes = [C.c_void_p, C.c_void_p]
    L.fe2_hrom_reset_points.argtypes = [C.c_void_p]
    L.fe2_hrom_snapshot.argtypes = [C.c_void_p]
    L.fe2_hrom_mono_begin.argtypes = [C.c_void_p]
    L.fe2_hrom_mono_iterate.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp, _ip, _ip]
    L.fe2_hrom_mono_commit.argtypes = [C.c_void_p]
    L.fe2_hrom_restore.argtypes = [C.c_void_p]
    L.fe2_hrom_output_ptrs.argtypes = [C.c_void_p] + [C.POINTER(C.c_void_p)] * 6
    L.fe2_nccl_get_unique_id.argtypes = [C.c_void_p]
    L.fe2_nccl_comm_init.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.POINTER(C.c_void_p)]
    L.fe2_nccl_comm_destroy.argtypes = [C.c_void_p]
    L.fe2_hrom_gather.argtypes = [C.c_void_p] * 6 + [C.c_double, C.c_void_p, _ip]
    L.fe2_hrom_gather_layout.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
    L.fe2_hrom_mono_iterate_device.argtypes = [C.c_void_p] * 8
    L.fe2_model_build.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, C.POINTER(C.c_void_p)]
    L.fe2_model_build_from_mesh.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_uint64, C.POINTER(C.c_void_p)]
    L.fe2_mesh_write.argtypes = [C.c_int, C.c_char_p]
    L.fe2_model_build_basis.argtypes = [C.c_int, C.c_char_p, _dp, C.c_int, C.c_int, C.c_uint64, C.POINTER(C.c_void_p)]
    L.fe2_hf_create.argtypes = [C.c_int, C.c_int, C.c_char_p, C.POINTER(_Material), C.c_int, C.POINTER(C.c_void_p)]
    L.fe2_hf_destroy.argtypes = [C.c_void_p]
    L.fe2_hf_destroy.restype = None
    L.fe2_hf_sizes.argtypes = [C.c_void_p, _ip, _ip, _ip, _dp]
    L.fe2_hf_trajectory.argtypes = [C.c_void_p, C.c_int, _dp, C.POINTER(_Opts), _dp, _dp, _ip, _dp, _dp, _dp]
    L.fe2_hf_elastic_modes.argtypes = [C.c_void_p, _dp, _ip]
    L.fe2_hf_trajectories.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp, C.POINTER(_Opts), _dp, _dp, _ip, _dp, _dp,
                                      _dp, _ip]
    L.fe2_hf_band.argtypes = [C.c_void_p, _ip]
    L.fe2_hrom_mixed_step.argtypes = [C.c_void_p, _ip, _dp, _dp, C.c_double, C.c_int, C.POINTER(_Opts), _dp, _dp,
                                      _dp, _ip, _ip]
    L.fe2_hf_mono_begin.argtypes = [C.c_void_p]
    L.fe2_hf_mono_iterate.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp, _ip]
    L.fe2_hf_mono_commit.argtypes = [C.c_void_p]
    L.fe2_hf_alloc_points.argtypes = [C.c_void_p, C.c_int64]
    L.fe2_hf_points.argtypes = [C.c_void_p, C.POINTER(C.c_int64)]
    L.fe2_hf_solve_increment.argtypes = [C.c_void_p, _dp, C.POINTER(_Opts), _dp, _dp, _ip, _ip]
    L.fe2_hf_snapshot.argtypes = [C.c_void_p]
    L.fe2_hf_restore.argtypes = [C.c_void_p]
    L.fe2_pod_basis.argtypes = [C.c_int, _dp, C.c_int64, C.c_int, _dp, C.c_int, C.c_int, _dp, _dp, _ip]
    L.fe2_model_free.argtypes = [C.c_void_p]
    L.fe2_model_free.restype = None
    L.fe2_model_sizes.argtypes = [C.c_void_p, _ip, _ip, _ip, _dp]
    L.fe2_model_arrays.argtypes = [C.c_void_p, _dp, _dp, _ip, _ip]
    L.fe2_paths.argtypes = [C.c_int, C.c_uint64, C.c_int64, C.c_int64, C.c_int, _dp]
    return L


lib = _load()


def _check(rc: int):
    if rc != 0:
        raise Fe2Error(rc, lib.fe2_last_error().decode())


def _d(a):
    return None if a is None else a.ctypes.data_as(_dp)


def _i(a):
    return None if a is None else a.ctypes.data_as(_ip)


def _u8(a):
    return None if a is None else a.ctypes.data_as(_u8p)


def device_count() -> int:
    return lib.fe2_device_count()


@dataclass
class ElasticParams:  # materials.hpp:37-43
    E: float = 1.0
    nu: float = 0.3

    def _c(self):
        return _Material(0, (C.c_double * 6)(self.E, self.nu, 0.0, 0.0, 0.0, 0.0))


@dataclass
class J2LinearParams:  # materials.hpp:45-49
    E: float = 1.0
    nu: float = 0.3
    sigma_y0: float = 0.01
    hardening: float = 0.016

    def _c(self):
        return _Material(1, (C.c_double * 6)(self.E, self.nu, self.sigma_y0, self.hardening, 0.0, 0.0))


@dataclass
class PowerLawParams:  # materials.hpp:51-65: sy(e) = sy0 (1 + E e / sy0)^N
    E: float = 1.0
    nu: float = 0.3
    sigma_y0: float = 0.01
    N: float = 0.1

    def _c(self):
        return _Material(2, (C.c_double * 6)(self.E, self.nu, self.sigma_y0, self.N, 0.0, 0.0))


@dataclass
class CreepParams:  # materials.hpp:67-76; dt = time of one load increment (PathStep::dt)
    E: float = 1.0
    nu: float = 0.14
    A: float = 22.09
    n: float = 1.06
    m: float = -0.56
    dt: float = 1.0

    def _c(self):
        return _Material(3, (C.c_double * 6)(self.E, self.nu, self.A, self.n, self.m, self.dt))


@dataclass
class NewtonOptions:  # MicroOptions rve.hpp:195-200 + TrajectoryOptions::max_bisections
    tol: float = 1e-8
    max_iter: int = 30
    max_bisections: int = 4

    def _c(self):
        return _Opts(self.tol, self.max_iter, self.max_bisections)


def update_material_batch(mat, eps, state=None, device=0):
    """Batched update_material on the GPU. eps (N,3) engineering Voigt,
    state (N,6) = (eps_p[4], eq, sigma33) or None (virgin).
    Returns sigma (N,3), C (N,3,3), state_out (N,6), plastic (N,) bool."""
    eps = np.ascontiguousarray(eps, dtype=np.float64).reshape(-1, 3)
    N = eps.shape[0]
    st = None if state is None else np.ascontiguousarray(state, dtype=np.float64).reshape(N, 6)
    sig = np.empty((N, 3))
    Cm = np.empty((N, 3, 3))
    so = np.empty((N, 6))
    pl = np.empty(N, dtype=np.uint8)
    m = mat._c()
    _check(lib.fe2_material_update_batch(device, C.byref(m), N, _d(eps), _d(st), _d(sig), _d(Cm), _d(so), _u8(pl)))
    return sig, Cm, so, pl.astype(bool)


def update_material_soa_device(mat, N, eps_ptr, hist_in_ptr, sigma_ptr, C6_ptr, hist_out_ptr=0, plastic_ptr=0,
                               stream=0, device=0):
    """Batched update_material on device SoA buffers (pointers as ints):
    eps[3][N], hist_in[5][N] (0 = virgin) -> sigma[3][N], C6[6][N]
    (C00 C01 C02 C11 C12 C22), hist_out[6][N], plastic[N] (u8). Async on stream."""
    m = mat._c()
    _check(lib.fe2_material_update_soa_device(device, C.byref(m), N, eps_ptr or None, hist_in_ptr or None,
                                              sigma_ptr or None, C6_ptr or None, hist_out_ptr or None,
                                              plastic_ptr or None, stream or None))


class HyperRomModel:
    """Offline stage: seeded hyper-ROM model on the default_cell RVE
    (mesh.hpp:185-191) — G[K,3,n], w[K], ip ids, material ids (0 matrix J2,
    1 inclusion), volume. Host only."""

    def __init__(self, subdivisions=33, n=12, K=200, seed=0, mesh_file: str | None = None, basis=None):
        """subdivisions: default_cell RVE; or mesh_file: an RVE in the
        reference's plain-text mesh format (write_mesh, mesh.hpp:413-489).
        basis: optional Φ (n, n_dofs) over all DOFs (e.g. pod.pod_basis)
        instead of the seeded orthonormal modes; n is then basis.shape[0]."""
        h = C.c_void_p()
        if basis is not None:
            basis = np.ascontiguousarray(basis, dtype=np.float64)
            n = basis.shape[0]
            path = None if mesh_file is None else str(mesh_file).encode()
            _check(lib.fe2_model_build_basis(subdivisions, path, _d(basis), n, K, seed, C.byref(h)))
        elif mesh_file is not None:
            _check(lib.fe2_model_build_from_mesh(str(mesh_file).encode(), n, K, seed, C.byref(h)))
        else:
            _check(lib.fe2_model_build(subdivisions, n, K, seed, C.byref(h)))
        try:
            n_, K_, nf, vol = C.c_int(), C.c_int(), C.c_int(), C.c_double()
            _check(lib.fe2_model_sizes(h, C.byref(n_), C.byref(K_), C.byref(nf), C.byref(vol)))
            self.n, self.K, self.n_free, self.volume = n_.value, K_.value, nf.value, vol.value
            self.G = np.empty((self.K, 3, self.n))
            self.w = np.empty(self.K)
            self.ip = np.empty(self.K, dtype=np.int32)
            self.mat = np.empty(self.K, dtype=np.int32)
            _check(lib.fe2_model_arrays(h, _d(self.G), _d(self.w), _i(self.ip), _i(self.mat)))
            self.G4 = np.empty((self.K, 4, self.n))  # displacement-gradient rows (finite strain)
            _check(lib.fe2_model_g4(h, _d(self.G4)))
        finally:
            lib.fe2_model_free(h)
        self.subdivisions, self.seed = subdivisions, seed
        self.materials = [J2LinearParams(1.0, 0.3, 0.01, 0.016), ElasticParams(10.0, 0.3)]

    @property
    def K_j2(self):
        return int(np.sum(self.mat == 0))


def write_mesh(subdivisions, path):
    """Write the default_cell(subdivisions) RVE in the reference's mesh format."""
    _check(lib.fe2_mesh_write(subdivisions, str(path).encode()))


def make_paths(kind, seed, P, n_incr, p0=0):
    """Seeded macro paths: kinds 0/1 (BASELINE configs 0/1) give strains
    E[P, n_incr, 3]; kind 2 (config 2) gives displacement gradients
    H[P, n_incr, 4] = (H00, H01, H10, H11), F = I + H."""
    E = np.empty((P, n_incr, 4 if kind == 2 else 3))
    _check(lib.fe2_paths(kind, seed, p0, P, n_incr, _d(E)))
    return E


def nccl_unique_id() -> bytes:
    """128-byte NCCL id (rank 0 makes it; broadcast it to the other ranks)."""
    buf = C.create_string_buffer(128)
    _check(lib.fe2_nccl_get_unique_id(buf))
    return buf.raw


class NcclComm:
    """One NCCL communicator per rank and device (fe2_nccl_comm_init)."""

    def __init__(self, device: int, nranks: int, rank: int, uid: bytes):
        assert len(uid) == 128
        self.nranks, self.rank = nranks, rank
        self._c = C.c_void_p()
        _check(lib.fe2_nccl_comm_init(device, nranks, rank, C.create_string_buffer(uid, 128), C.byref(self._c)))

    @property
    def ptr(self):
        return self._c.value

    def close(self):
        if self._c.value:
            _check(lib.fe2_nccl_comm_destroy(self._c))
            self._c = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class HyperRomEngine:
    """One device's batch of macro Gauss points evaluated with a hyper-ROM
    RVE model: the reduced form of run_trajectory (rve.hpp:448-494) per
    point, one increment per call.

    Small strain (G[K,3,n]): inputs E (P,3), outputs sigma (P,3), C (P,3,3).
    Finite strain (G[K,4,n], Biot J2, BASELINE config 2): inputs H = F - I
    (P,4), outputs under the same keys: sigma = P_M (P,4) first
    Piola-Kirchhoff stress, C = A_M (P,4,4) = dP_M/dF."""

    def __init__(self, G, w, mat_id, materials, volume, device=0):
        G = np.ascontiguousarray(G, dtype=np.float64)
        K, rows, n = G.shape
        assert rows in (3, 4)
        self.n, self.K = n, K
        self.finite = rows == 4
        self.nc = rows
        self._w = np.ascontiguousarray(w, dtype=np.float64)
        self._mid = np.ascontiguousarray(mat_id, dtype=np.int32)
        mats = (_Material * len(materials))(*[m._c() for m in materials])
        h = C.c_void_p()
        create = lib.fe2_hrom_create_fs if self.finite else lib.fe2_hrom_create
        _check(create(device, n, K, _d(G), _d(self._w), _i(self._mid), mats, len(materials), float(volume),
                      C.byref(h)))
        self._h = h
        self.P = 0

    @classmethod
    def from_model(cls, model: HyperRomModel, device=0, finite_strain=False):
        G = model.G4 if finite_strain else model.G
        return cls(G, model.w, model.mat, model.materials, model.volume, device)

    def close(self):
        if getattr(self, "_h", None):
            lib.fe2_hrom_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def alloc_points(self, P, keep_flags=False):
        _check(lib.fe2_hrom_alloc_points(self._h, P, 1 if keep_flags else 0))
        self.P = P

    def reset_points(self):
        _check(lib.fe2_hrom_reset_points(self._h))

    def snapshot(self):
        """Save the committed state of every point (deferred-commit callers)."""
        _check(lib.fe2_hrom_snapshot(self._h))

    def restore(self):
        """Return every point to the last snapshot."""
        _check(lib.fe2_hrom_restore(self._h))

    def mono_begin(self):
        """Monolithic scheme: start a step from the committed state."""
        _check(lib.fe2_hrom_mono_begin(self._h))

    def mono_iterate(self, E):
        """One monolithic micro iteration of every point at macro strains E
        (P,3): condensed sigma (P,3), C (P,3,3), rel_res, plastic_count, status."""
        E = np.ascontiguousarray(E, dtype=np.float64).reshape(self.P, 3)
        sig, Cm, rr = np.empty((self.P, 3)), np.empty((self.P, 3, 3)), np.empty(self.P)
        pc, st = np.empty(self.P, dtype=np.int32), np.empty(self.P, dtype=np.int32)
        _check(lib.fe2_hrom_mono_iterate(self._h, _d(E), _d(sig), _d(Cm), _d(rr), _i(pc), _i(st)))
        return dict(sigma=sig, C=Cm, rel_res=rr, plastic_count=pc, status=st)

    def mono_commit(self):
        """Adopt the last monolithic iterate of every point as committed."""
        _check(lib.fe2_hrom_mono_commit(self._h))

    def output_ptrs(self):
        """Device pointers (ints) of the handle's own output buffers:
        sigma, C, iters, plastic_count, res_norm, status."""
        ps = [C.c_void_p() for _ in range(6)]
        _check(lib.fe2_hrom_output_ptrs(self._h, *[C.byref(p) for p in ps]))
        return [p.value for p in ps]

    def gather_layout(self, comm: "NcclComm"):
        """fe2_hrom_gather_layout: (P_max, per-rank point counts) over comm; the
        gathered buffer holds world blocks of P_max rows (padding: status -1)."""
        pmax = C.c_int64()
        counts = (C.c_int64 * comm.nranks)()
        _check(lib.fe2_hrom_gather_layout(self._h, comm.ptr, C.byref(pmax), counts))
        return pmax.value, list(counts)

    def gather(self, comm: "NcclComm", d_all: int, sigma=0, Cm=0, res=0, status=0, res_tol=float("inf"),
               flags=False, wait=True):
        """fe2_hrom_gather: all-gather every rank's records {Σ | C | ‖r‖ |
        status} of the last increment / monolithic iterate into the device
        buffer d_all ([world][P_max][nc + nt + 2] doubles) over NCCL; the
        device outputs default to the handle's own buffers. Returns the
        all-reduced "some point failed" flag, or with flags=True the pair
        (some point failed, some point has ‖r‖ > res_tol); wait=False keeps
        the call asynchronous (returns None)."""
        fl = np.zeros(2, dtype=np.int32)
        _check(lib.fe2_hrom_gather(self._h, comm.ptr, sigma or None, Cm or None, res or None, status or None,
                                   float(res_tol), d_all, _i(fl) if wait else None))
        if not wait:
            return None
        return (bool(fl[0]), bool(fl[1])) if flags else bool(fl[0])

    def mono_iterate_device(self, E_ptr, sigma=0, Cm=0, rel_res=0, pc=0, status=0, stream=0):
        """fe2_hrom_mono_iterate_device: one monolithic iteration at the macro
        strains E_ptr (device, P x 3), asynchronous; NULL outputs = the handle's."""
        _check(lib.fe2_hrom_mono_iterate_device(self._h, E_ptr, sigma or None, Cm or None, rel_res or None,
                                                pc or None, status or None, stream or None))

    def solve_increment_into(self, E, sigma, Cm, iters, pc, res, status, opts: NewtonOptions | None = None):
        """Host-buffer C-ABI call writing into caller-provided (e.g. pinned)
        numpy arrays; E (P,3) host."""
        o = (opts or NewtonOptions())._c()
        _check(lib.fe2_hrom_solve_increment(self._h, _d(E), C.byref(o), _d(sigma), _d(Cm), _i(iters), _i(pc),
                                            _d(res), _i(status)))

    def solve_increment_async_into(self, E, sigma, Cm, iters, pc, res, status, opts: NewtonOptions | None = None):
        """Queue one increment (host buffers, pinned for overlap); the outputs
        are written asynchronously — valid after wait()."""
        o = (opts or NewtonOptions())._c()
        _check(lib.fe2_hrom_solve_increment_async(self._h, _d(E), C.byref(o), _d(sigma), _d(Cm), _i(iters), _i(pc),
                                                  _d(res), _i(status)))

    def wait(self):
        """Wait for all queued asynchronous increments and their output copies."""
        _check(lib.fe2_hrom_wait(self._h))

    def solve_increment(self, E, opts: NewtonOptions | None = None):
        """E (P,3) host → dict of sigma (P,3), C (P,3,3), iters, plastic_count, res_norm, status.
        (finite strain: H (P,4) → sigma = P_M (P,4), C = A_M (P,4,4))"""
        nc = self.nc
        E = np.ascontiguousarray(E, dtype=np.float64).reshape(self.P, nc)
        out = dict(
            sigma=np.empty((self.P, nc)), C=np.empty((self.P, nc, nc)), iters=np.empty(self.P, dtype=np.int32),
            plastic_count=np.empty(self.P, dtype=np.int32), res_norm=np.empty(self.P),
            status=np.empty(self.P, dtype=np.int32))
        o = (opts or NewtonOptions())._c()
        _check(lib.fe2_hrom_solve_increment(self._h, _d(E), C.byref(o), _d(out["sigma"]), _d(out["C"]),
                                            _i(out["iters"]), _i(out["plastic_count"]), _d(out["res_norm"]),
                                            _i(out["status"])))
        return out

    def solve_increment_device(self, E_ptr, sigma_ptr, C_ptr, iters_ptr, pc_ptr, res_ptr, status_ptr, stream=0,
                               opts: NewtonOptions | None = None):
        """Device-pointer variant (inputs already resident in HBM)."""
        o = (opts or NewtonOptions())._c()
        _check(lib.fe2_hrom_solve_increment_device(self._h, E_ptr, C.byref(o), sigma_ptr, C_ptr, iters_ptr, pc_ptr,
                                                   res_ptr, status_ptr, stream or None))

    def read_state(self, flags=False):
        alpha = np.empty((self.P, self.n))
        state = np.empty((self.P, self.K, 6))
        fl = np.empty((self.P, self.K), dtype=np.uint8) if flags else None
        _check(lib.fe2_hrom_read_state(self._h, _d(alpha), _d(state), _u8(fl)))
        return alpha, state, fl

    def assemble_point(self, point, alpha, E):
        n = self.n
        r, Kaa, KaE = np.empty(n), np.empty((n, n)), np.empty((n, 3))
        CEE, S = np.empty((3, 3)), np.empty(3)
        alpha = np.ascontiguousarray(alpha, dtype=np.float64)
        E = np.ascontiguousarray(E, dtype=np.float64)
        _check(lib.fe2_hrom_assemble_point(self._h, point, _d(alpha), _d(E), _d(r), _d(Kaa), _d(KaE), _d(CEE),
                                           _d(S)))
        return dict(r=r, Kaa=Kaa, KaE=KaE, C_EE=CEE, S_raw=S)

    def fs_assemble_point(self, point, alpha, H):
        """Finite-strain assembly of a point's committed history at (alpha, H)."""
        n = self.n
        r, Kaa, KaF, KFa = np.empty(n), np.empty((n, n)), np.empty((n, 4)), np.empty((4, n))
        CFF, Praw = np.empty((4, 4)), np.empty(4)
        alpha = np.ascontiguousarray(alpha, dtype=np.float64)
        H = np.ascontiguousarray(H, dtype=np.float64)
        _check(lib.fe2_hrom_fs_assemble_point(self._h, point, _d(alpha), _d(H), _d(r), _d(Kaa), _d(KaF), _d(KFa),
                                              _d(CFF), _d(Praw)))
        return dict(r=r, Kaa=Kaa, KaF=KaF, KFa=KFa, C_FF=CFF, P_raw=Praw)

    def stats(self):
        s = _Stats()
        _check(lib.fe2_hrom_stats(self._h, C.byref(s)))
        return {k: getattr(s, k) for k, _ in s._fields_}

    def set_timing(self, on=True):
        _check(lib.fe2_hrom_set_timing(self._h, 1 if on else 0))

    def reset_stats(self):
        _check(lib.fe2_hrom_reset_stats(self._h))

    def mixed_step(self, control, E_prescribed, sigma_target, E, tol=1e-10, max_iter=25,
                   opts: NewtonOptions | None = None):
        """Mixed control for every point (fe2_hrom_mixed_step; rve.hpp:496-571):
        control (P,3) bool (True = strain prescribed), E_prescribed / sigma_target
        (P,3); E (P,3) the committed macro strains. Returns E (converged), sigma,
        C (P,3,3), outer_iters, status; the engine is left at the accepted state."""
        P = self.P
        ctl = np.ascontiguousarray(np.broadcast_to(np.asarray(control, dtype=np.int32), (P, 3)))
        Ep = np.ascontiguousarray(np.broadcast_to(np.asarray(E_prescribed, dtype=np.float64), (P, 3)))
        St = np.ascontiguousarray(np.broadcast_to(np.asarray(sigma_target, dtype=np.float64), (P, 3)))
        Eo = np.array(np.broadcast_to(np.asarray(E, dtype=np.float64), (P, 3)))
        sig, Cm = np.empty((P, 3)), np.empty((P, 3, 3))
        it, st = np.empty(P, dtype=np.int32), np.empty(P, dtype=np.int32)
        o = (opts or NewtonOptions())._c()
        _check(lib.fe2_hrom_mixed_step(self._h, _i(ctl), _d(Ep), _d(St), tol, max_iter, C.byref(o), _d(Eo), _d(sig),
                                       _d(Cm), _i(it), _i(st)))
        return dict(E=Eo, sigma=sig, C=Cm, outer_iters=it, status=st)

    def set_stream(self, stream_ptr):
        """Order the engine's work on a caller's cudaStream_t (int handle; 0 = own)."""
        _check(lib.fe2_hrom_set_stream(self._h, stream_ptr or None))
