"""Build the in-tree CUDA library `libbddc_b200.so` for sm_100a.

nvcc compiles the device kernels (-gencode arch=compute_100a,code=sm_100a,
-lineinfo) and the C++ host layer; the shared library is written next to
this file so it travels with the repo snapshot to the GPU box.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
CSRC = HERE / "csrc"
LIB = HERE / "libbddc_b200.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
          "-Xcompiler", "-fopenmp", "-I", str(HERE.parent / "include")]


def sources():
    return sorted(list((CSRC / "cuda").glob("*.cu")) + list((CSRC / "host").glob("*.cpp")) +
                  [CSRC / "capi.cpp"])


def headers():
    return sorted(list(CSRC.rglob("*.hpp")) + list(CSRC.rglob("*.cuh")) +
                  [HERE.parent / "include" / "bddc_b200.h"])


def build(force: bool = False, verbose: bool = False) -> Path:
    srcs = sources()
    newest = max(p.stat().st_mtime for p in srcs + headers())
    if LIB.exists() and not force and LIB.stat().st_mtime >= newest:
        return LIB
    objdir = HERE / "build"
    objdir.mkdir(exist_ok=True)
    objs = []
    procs = []
    for src in srcs:
        obj = objdir / (src.stem + (".cu.o" if src.suffix == ".cu" else ".o"))
        cmd = [NVCC, *ARCH, *COMMON, "-c", str(src), "-o", str(obj)]
        if src.suffix == ".cu":
            cmd += ["-Xptxas", "-v"] if verbose else []
        else:
            cmd += ["-x", "c++"]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    failed = False
    for src, p in procs:
        out = p.communicate()[0].decode()
        if p.returncode != 0:
            failed = True
            sys.stderr.write("nvcc failed for %s:\n%s\n" % (src, out))
        elif verbose and out.strip():
            sys.stderr.write(out)
    if failed:
        raise RuntimeError("CUDA build failed")
    tmp = LIB.with_suffix(".so.tmp")
    subprocess.check_call([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(tmp), *map(str, objs),
                           "-lgomp", "-ldl"])
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
