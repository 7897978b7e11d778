"""Build recipe for the native engine (sm_100a).

libfe2rom_gpu.so = C-ABI host driver + sm_100a kernels + offline setup,
built in-tree with nvcc so the .so travels with the repo snapshot.
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "lib", "libfe2rom_gpu.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
SOURCES = ["hrom_host.cu", "hrom_kernels.cu", "hrom_kernels_big.cu", "hrom_kernels_big_mono.cu", "hrom_kernels_big_other.cu", "hrom_kernels_big_gen.cu", "hrom_kernels_fs.cu", "material_soa.cu", "setup.cpp", "macro.cpp", "ecm.cpp", "hf.cu", "exchange.cu"]
HEADERS = ["common.hpp", "material.cuh", "hrom_kernels.cuh", "device_common.cuh", "biot.cuh", "host_util.cuh", "rve.hpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++20", "-Xcompiler", "-fPIC,-ffp-contract=off",
         "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src, obj, defines):
    cmd = [NVCC, *ARCH, *FLAGS, *[f"-D{d}" for d in defines], "-c", "-I", os.path.join(ROOT, "include"),
           "-I", CSRC, "-o", obj, os.path.join(CSRC, src)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    return src, r.returncode, r.stdout + r.stderr


def build_native(force=False, verbose=False, out=None, defines=()):
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "fe2rom", "fe2rom_gpu.h"))
    deps.append(os.path.abspath(__file__))
    target = out or LIB
    if not force and not _stale(target, deps):
        return target
    os.makedirs(os.path.dirname(target), exist_ok=True)
    # one nvcc per translation unit, in parallel, then one link
    from concurrent.futures import ThreadPoolExecutor
    objdir = target + ".obj"
    os.makedirs(objdir, exist_ok=True)
    objs = [os.path.join(objdir, s + ".o") for s in SOURCES]
    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 4)) as ex:
        results = list(ex.map(lambda so: _compile(so[0], so[1], defines), zip(SOURCES, objs)))
    log = "".join(f"==== {src}\n{txt}" for src, _, txt in results)
    failed = [src for src, rc, _ in results if rc != 0]
    if failed:
        sys.stderr.write(log)
        raise RuntimeError(f"nvcc build of libfe2rom_gpu.so failed ({', '.join(failed)})")
    r = subprocess.run([NVCC, *ARCH, "-shared", "-o", target + ".tmp", *objs, "-ldl"], capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link of libfe2rom_gpu.so failed")
    with open(target + ".ptxas.log", "w") as f:
        f.write(log)
    if verbose:
        sys.stderr.write(log)
    os.replace(target + ".tmp", target)
    return target


if __name__ == "__main__":
    # python build.py [--force] [--variant NAME D1=V1 D2=V2 ...]  (variants go to lib/variants/)
    if "--variant" in sys.argv:
        i = sys.argv.index("--variant")
        name, defs = sys.argv[i + 1], sys.argv[i + 2:]
        print(build_native(force=True, out=os.path.join(HERE, "lib", "variants", f"lib_{name}.so"), defines=defs))
    else:
        print(build_native(force="--force" in sys.argv, verbose=True))
