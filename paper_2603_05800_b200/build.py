"""Build libsw_plan.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libsw_plan.so")
INCLUDE = os.path.join(ROOT, "include")


def nccl_paths():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    cands = []
    if spec and spec.submodule_search_locations:
        for loc in spec.submodule_search_locations:
            cands.append(os.path.join(loc, "nccl"))
    for c in cands:
        if os.path.exists(os.path.join(c, "include", "nccl.h")):
            return os.path.join(c, "include"), os.path.join(c, "lib")
    raise RuntimeError("nccl.h not found (expected the torch-bundled nvidia/nccl)")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                  + [os.path.join(INCLUDE, "sw_plan.h")])


STAMP = LIB + ".sha256"  # hash of the sources the library was built from


def source_hash() -> str:
    import hashlib
    h = hashlib.sha256()
    for s in sources():
        h.update(os.path.basename(s).encode())
        with open(s, "rb") as f:
            h.update(f.read())
    return h.hexdigest()


def needs_build() -> bool:
    """True when the library is missing or was built from other sources (content hash,
    so a snapshot copied to another box with fresh mtimes is still recognised)."""
    if not os.path.exists(LIB) or not os.path.exists(STAMP):
        return True
    with open(STAMP) as f:
        return f.read().strip() != source_hash()


def build(force: bool = False, verbose: bool = False, out: str = None, defines=()) -> str:
    """Compile libsw_plan.so (out/defines: experiment variants, tools/build_variant.py)."""
    if out is None and not force and not needs_build():
        return LIB
    inc, lib = nccl_paths()
    src_hash = source_hash()  # of the sources as they are when the compile starts
    cmd = [
        "nvcc", "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
        "-Xcompiler", "-fPIC", "-shared",
        "-Xptxas", "-v" if verbose else "-O3",
        "-I", INCLUDE, "-I", inc, "-cudart", "static",
        "-DSW_BUILD_SHARED", *["-D" + d for d in defines],
        os.path.join(CSRC, "sw_plan.cu"),
        "-L", lib, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + lib,
        "-o", out or LIB,
    ]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed")
    if verbose:
        sys.stderr.write(r.stderr)
    if out:
        return out
    with open(STAMP, "w") as f:
        f.write(src_hash + "\n")
    return LIB


if __name__ == "__main__":
    build(force=True, verbose="-v" in sys.argv)
    print(LIB)
