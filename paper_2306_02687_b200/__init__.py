"""fe2rom-b200: B200-native online hot path of the monolithic hyper-ROM FE²
method (arXiv 2306.02687) — batched evaluation of hyper-reduced RVE models at
every macro Gauss point.

The compute path is the native library ``lib/libfe2rom_gpu.so`` (C ABI in
``include/fe2rom/fe2rom_gpu.h``; sm_100a kernels). This package is the thin
Python mirror of the reference's material-point and solver interface
(``/root/reference/proj/include/fe2rom``: ``update_material``,
``micro_newton``/``homogenize``/``run_trajectory``) over that ABI. There is
no CPU fallback: without the library or a B200, calls raise.
"""
from .hrom import (  # noqa: F401
    CreepParams,
    ElasticParams,
    Fe2Error,
    HyperRomEngine,
    HyperRomModel,
    J2LinearParams,
    NewtonOptions,
    PowerLawParams,
    device_count,
    NcclComm,
    lib,
    nccl_unique_id,
    make_paths,
    update_material_batch,
    write_mesh,
    update_material_soa_device,
)
from .fe2 import MacroConfig, macro_gauss, macro_points, solve_program  # noqa: F401
from .pod import HfRve, pod_basis  # noqa: F401

__all__ = [
    "CreepParams",
    "PowerLawParams",
    "ElasticParams",
    "Fe2Error",
    "HyperRomEngine",
    "HyperRomModel",
    "J2LinearParams",
    "NewtonOptions",
    "device_count",
    "lib",
    "make_paths",
    "write_mesh",
    "update_material_batch",
    "update_material_soa_device",
    "MacroConfig",
    "macro_gauss",
    "macro_points",
    "solve_program",
    "HfRve",
    "pod_basis",
]
