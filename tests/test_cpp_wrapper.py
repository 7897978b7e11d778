"""The C++ host mirror (include/fe2rom/hrom_gpu.hpp) compiles against the
C ABI and links the in-tree library; without a GPU it raises the reference
Error with ErrorCode::numeric (no CPU fallback); with one it runs."""
import os
import subprocess

import pytest

import paper_2306_02687_b200 as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def build_example(tmp_path):
    exe = str(tmp_path / "hrom_cpp_example")
    libdir = os.path.dirname(F.hrom.LIB_PATH)
    cmd = ["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "examples",
           "hrom_cpp_example.cpp"), "-L", libdir, "-lfe2rom_gpu", f"-Wl,-rpath,{libdir}", "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True)
    return exe


def test_cpp_wrapper_builds_and_reports(tmp_path):
    exe = build_example(tmp_path)
    r = subprocess.run([exe, "3"], capture_output=True, text=True, timeout=120)
    if F.device_count() == 0:
        assert r.returncode == 2 and "no CUDA device" in r.stdout
    else:
        assert r.returncode == 0 and "increment 5 point 0" in r.stdout


@pytest.mark.gpu
def test_cpp_wrapper_runs_on_gpu(tmp_path):
    """The C++ mirror's numbers against the oracle: config-0 model, 8 points x 5
    increments, small strain (Σ, C_macro, iterations) and finite strain (P_M, A_M)."""
    import numpy as np
    import pyoracle as O
    from test_gpu_parity import REL, rel_err
    exe = build_example(tmp_path)
    P, n_incr = 8, 5
    r = subprocess.run([exe, str(P)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("finite-strain increment") == 5
    rows = {"R": {}, "F": {}}
    for ln in r.stdout.splitlines():
        f = ln.split()
        if f and f[0] in rows:
            rows[f[0]][(int(f[1]), int(f[2]))] = (int(f[3]), np.array([float(x) for x in f[4:]]))
    assert len(rows["R"]) == len(rows["F"]) == P * n_incr
    m = F.HyperRomModel(33, 12, 200, 0)
    o = O.Hrom(m.G, m.w, m.mat, m.materials, m.volume).run(F.make_paths(0, 0, P, n_incr))
    ofs = O.HromFs(m.G4, m.w, m.mat, m.materials, m.volume).run(F.make_paths(2, 0, P, n_incr))
    for (k, p), (it, v) in rows["R"].items():
        assert it == o["iters"][p, k]
        assert rel_err(v[None, :3], o["sigma"][p, k][None]).max() < REL
        assert rel_err(v[None, 3:], o["C"][p, k].reshape(1, 9)).max() < REL
    for (k, p), (it, v) in rows["F"].items():
        assert it == ofs["iters"][p, k]
        assert rel_err(v[None, :4], ofs["P"][p, k][None]).max() < REL
        assert rel_err(v[None, 4:], ofs["A"][p, k].reshape(1, 16)).max() < REL
