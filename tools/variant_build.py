#!/usr/bin/env python
"""Builds a product-flag variant of the library with extra -D definitions (A/B measurements, not shipped):
    python tools/variant_build.py -DLARS_SQ8_F32=0   ->  build/variants/liblars_LARS_SQ8_F32_0.so
Load it with LARS_LIB=<path> (tools/knob_sweep.py, bench.py and the tests honour it)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1903_12650_b200 import build as B  # noqa: E402

defs = [a for a in sys.argv[1:] if a.startswith("-D")]
tag = "_".join(d[2:].replace("=", "_") for d in defs) or "base"
out = os.path.join(ROOT, "build", "variants", tag)
os.makedirs(out, exist_ok=True)
nccl = B.nccl_root()
objs = []
for src in B.sources():
    obj = os.path.join(out, os.path.basename(src) + ".o")
    subprocess.check_call([B.NVCC, *B.ARCH, "-O3", "-std=c++17", "-lineinfo", *defs, "-Xcompiler", "-fPIC",
                           "-I", os.path.join(ROOT, "include"), "-I", B.CSRC, "-I", os.path.join(nccl, "include"),
                           "-c", src, "-o", obj])
    objs.append(obj)
lib = os.path.join(ROOT, "build", "variants", f"liblars_{tag}.so")
subprocess.check_call([B.NVCC, *B.ARCH, "-shared", "-cudart", "static", "-o", lib, *objs, "-L",
                       os.path.join(nccl, "lib"), "-l:libnccl.so.2", "-Xlinker", f"-rpath,{os.path.join(nccl, 'lib')}"])
print(lib)
