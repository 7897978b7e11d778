"""Regenerate tests/golden/ from the REFERENCE's own code (test infrastructure).

Runs oracle/_ref/ref_golden (the reference headers compiled unmodified against the
Eigen-API shim, `make -C oracle ref`) and writes:
  tests/golden/ref_*.npy         small fixtures (materials, default_cell(6/8) meshes, HF runs)
  tests/golden/ref_manifest.json sha256 of every fixture + of the default_cell(33) mesh
                                 arrays (too large to commit; tests hash their own copy)
                                 + sha256 of the reference headers they came from.
Only usable where /root/reference exists (the build container).
"""
import glob
import hashlib
import json
import os
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
GOLD = os.path.join(ROOT, "tests", "golden")
REF = "/root/reference/proj"


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)
    exe = os.path.join(HERE, "_ref", "ref_golden")
    os.makedirs(GOLD, exist_ok=True)
    for f in glob.glob(os.path.join(GOLD, "ref_*")):
        os.remove(f)
    manifest = {"generator": "oracle/ref_golden.cpp via oracle/make_golden.py",
                "reference_headers": {}, "fixtures": {}, "mesh33": {}}
    for h in sorted(glob.glob(os.path.join(REF, "include", "fe2rom", "*.hpp"))):
        manifest["reference_headers"][os.path.relpath(h, "/root/reference")] = hashlib.sha256(open(h, "rb").read()).hexdigest()
    with tempfile.TemporaryDirectory() as td:
        subprocess.run([exe, td], check=True)
        for f in sorted(os.listdir(td)):
            if f.endswith(".txt"):
                data = open(os.path.join(td, f), "rb").read()
                open(os.path.join(GOLD, "ref_" + f), "wb").write(data)
                manifest["fixtures"]["ref_" + f] = {"bytes": len(data), "sha256": hashlib.sha256(data).hexdigest()}
                continue
            a = np.load(os.path.join(td, f))
            np.save(os.path.join(GOLD, "ref_" + f), a)
            manifest["fixtures"]["ref_" + f] = {"shape": list(a.shape), "sha256": sha(a)}
        subprocess.run([exe, td, "--big"], check=True)
        for part in ("xy", "conn", "ip", "meta"):
            a = np.load(os.path.join(td, f"mesh33_{part}.npy"))
            manifest["mesh33"][part] = {"shape": list(a.shape), "dtype": str(a.dtype), "sha256": sha(a)}
        data = open(os.path.join(td, "mesh33_text.txt"), "rb").read()
        manifest["mesh33"]["text"] = {"bytes": len(data), "sha256": hashlib.sha256(data).hexdigest()}
    with open(os.path.join(GOLD, "ref_manifest.json"), "w") as f:
        json.dump(manifest, f, indent=1)
    print(f"wrote {len(manifest['fixtures'])} fixtures to {GOLD}")


if __name__ == "__main__":
    sys.exit(main())
