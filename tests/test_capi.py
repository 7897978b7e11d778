"""The drop-in boundary: the C-ABI library loads, exports every entry point
declared in include/fe2rom/fe2rom_gpu.h, validates arguments with the
reference error taxonomy, and fails loudly (no CPU fallback) without a GPU."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2306_02687_b200 as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fe2rom", "fe2rom_gpu.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fe2_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(F.hrom.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_version_and_device_count():
    assert b"sm_100a" in F.lib.fe2_version()
    assert F.device_count() >= 0


def test_invalid_arguments_use_reference_error_codes():
    m = F.HyperRomModel(8, 6, 40, 0)
    with pytest.raises(F.Fe2Error) as e:  # materials.hpp:80-82 validate -> ErrorCode::config
        F.HyperRomEngine(m.G, m.w, m.mat, [F.J2LinearParams(E=-1.0), F.ElasticParams()], m.volume)
    assert e.value.kind == "config"
    with pytest.raises(F.Fe2Error) as e:
        F.HyperRomModel(33, 0, 10, 0)
    assert e.value.kind == "config"
    with pytest.raises(F.Fe2Error) as e:  # mesh.hpp:196-210 geometry validation
        F.HyperRomModel(5, 4, 10, 0)
    assert e.value.kind == "geometry"


@pytest.mark.skipif(F.device_count() > 0, reason="checks the no-GPU behaviour")
def test_no_cpu_fallback_without_gpu():
    m = F.HyperRomModel(8, 6, 40, 0)
    with pytest.raises(F.Fe2Error) as e:
        F.HyperRomEngine.from_model(m)
    assert e.value.kind == "numeric" and "no CPU fallback" in str(e.value)
    with pytest.raises(F.Fe2Error):
        F.update_material_batch(F.J2LinearParams(), np.zeros((4, 3)))


def test_oracle_header_is_test_infrastructure_only():
    """The product package never imports the oracle."""
    pkg = os.path.join(ROOT, "paper_2306_02687_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".hpp", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f), encoding="utf-8").read()
                assert "pyoracle" not in txt and "fe2rom_oracle" not in txt and "liboracle" not in txt, f


def test_exchange_entry_points_validate_and_need_a_device():
    """fe2_hrom_gather / fe2_nccl_comm_init: argument checks
    with the reference taxonomy; no communicator without a CUDA device."""
    flag = np.zeros(2, dtype=np.int32)
    rc = F.lib.fe2_hrom_gather(None, None, None, None, None, None, 0.0, None,
                               flag.ctypes.data_as(ctypes.POINTER(ctypes.c_int)))
    assert rc == 1  # ErrorCode::config ("no points allocated")
    rc = F.lib.fe2_hrom_gather_layout(None, None, None, None)
    assert rc == 1
    out = ctypes.c_void_p()
    rc = F.lib.fe2_nccl_comm_init(0, 2, 5, ctypes.create_string_buffer(128), ctypes.byref(out))
    assert rc == 1  # rank out of range -> config
    if F.device_count() == 0:
        with pytest.raises(F.Fe2Error) as e:
            F.NcclComm(0, 1, 0, bytes(128))
        assert e.value.kind == "numeric" and "no CPU fallback" in str(e.value)


def test_round2_entry_points_validate_arguments():
    """fe2_hrom_mixed_step, fe2_hf_trajectories / _mono_* / _band: null handles and
    bad options return ErrorCode::config (1) without touching a device."""
    o = F.hrom.NewtonOptions()._c()
    assert F.lib.fe2_hrom_mixed_step(None, None, None, None, 1e-10, 25, ctypes.byref(o), None, None, None, None,
                                     None) == 1
    assert F.lib.fe2_hf_trajectories(None, 1, 1, None, ctypes.byref(o), None, None, None, None, None, None,
                                     None) == 1
    assert F.lib.fe2_hf_mono_begin(None) == 1
    assert F.lib.fe2_hf_mono_commit(None) == 1
    assert F.lib.fe2_hf_mono_iterate(None, None, None, None, None, None) == 1
    b = ctypes.c_int()
    assert F.lib.fe2_hf_band(None, ctypes.byref(b)) == 1
