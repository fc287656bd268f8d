"""Builds the in-tree C-ABI library ``paper_1903_12650_b200/liblars_b200.so`` for sm_100a.

nvcc cross-compiles without a GPU. NCCL is torch's own copy (pip ``nvidia-nccl-cu12``, 2.28.x) so
that exactly one NCCL is loaded per process; the CUDA runtime is linked statically.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build")
LIB = os.path.join(PKG, "liblars_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_root() -> str:
    for p in sys.path:
        cand = os.path.join(p, "nvidia", "nccl")
        if os.path.exists(os.path.join(cand, "include", "nccl.h")):
            return cand
    raise RuntimeError("torch's NCCL (nvidia/nccl/include/nccl.h) not found on sys.path")


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.h")) + [os.path.join(ROOT, "include", "lars.h"), __file__]
    return any(os.path.getmtime(d) > t for d in deps)


CHECKED_LIB = os.path.join(BUILD, "checked", "liblars_b200_checked.so")


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    """checked=True: the diagnostics variant with device-side bounds/invariant checks (-DLARS_DEVICE_CHECKS),
    written to build/checked/ (never the in-tree product library); load it with LARS_LIB=<path>."""
    lib = CHECKED_LIB if checked else LIB
    if not force and not checked and not _stale():
        return LIB
    nccl = nccl_root()
    build_dir = os.path.join(BUILD, "checked") if checked else BUILD
    os.makedirs(build_dir, exist_ok=True)
    common = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-Wall", "-I", os.path.join(ROOT, "include"),
              "-I", CSRC, "-I", os.path.join(nccl, "include")] + (["-DLARS_DEVICE_CHECKS"] if checked else [])
    objs = []
    for src in sources():
        obj = os.path.join(build_dir, os.path.basename(src) + ".o")
        cmd = [NVCC, *ARCH, *common, "-c", src, "-o", obj]
        if src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        if verbose and r.stderr:
            print(r.stderr, file=sys.stderr)
        if src.endswith(".cu"):
            with open(os.path.join(build_dir, "ptxas.log"), "w") as f:
                f.write(r.stderr)
        objs.append(obj)
    libdir = os.path.join(nccl, "lib")
    tmp = lib + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs, "-L", libdir, "-l:libnccl.so.2",
           "-Xlinker", f"-rpath,{libdir}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, checked="--checked" in sys.argv))
