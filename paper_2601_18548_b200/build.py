"""Build libgcdf.so in-tree with nvcc for sm_100a (B200).

    python -m paper_2601_18548_b200.build [--force] [--verbose]

Every .cu / .cpp under csrc/ is compiled with
-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo and linked into
paper_2601_18548_b200/libgcdf.so (CUDA runtime linked statically).
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libgcdf.so"
OBJ = PKG.parent / "build" / "obj"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
         "--expt-relaxed-constexpr", "-I", str(PKG.parent / "include")]


def sources():
    return sorted(list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cpp")))


def build(force: bool = False, verbose: bool = False) -> str:
    OBJ.mkdir(parents=True, exist_ok=True)
    headers = list(CSRC.glob("*.h")) + list((PKG.parent / "include").glob("*.h"))
    hmax = max((h.stat().st_mtime for h in headers), default=0)
    objs = []
    for src in sources():
        obj = OBJ / (src.name + ".o")
        objs.append(obj)
        if force or not obj.exists() or obj.stat().st_mtime < max(src.stat().st_mtime, hmax):
            cmd = [NVCC, *ARCH, *FLAGS, "-c", str(src), "-o", str(obj)]
            if verbose and src.suffix == ".cu":
                cmd += ["-Xptxas", "-v"]
            print(" ".join(cmd), file=sys.stderr, flush=True)
            subprocess.check_call(cmd)
    if force or not LIB.exists() or LIB.stat().st_mtime < max(o.stat().st_mtime for o in objs):
        tmp = LIB.with_suffix(".so.tmp%d" % os.getpid())
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(tmp), *map(str, objs)]
        print(" ".join(cmd), file=sys.stderr, flush=True)
        subprocess.check_call(cmd)
        os.replace(tmp, LIB)
    return str(LIB)


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="--verbose" in sys.argv)
