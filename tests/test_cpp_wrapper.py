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
    exe = build_example(tmp_path)
    r = subprocess.run([exe, "8"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("finite-strain increment") == 5
    assert r.stdout.count("increment") == 10
