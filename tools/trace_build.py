#!/usr/bin/env python
"""Builds the diagnostics variant build/liblars_trace.so (kernels compiled with -DLARS_TRACE: per-CTA
start/end %globaltimer + %smid). Not the product library; used by tools/trace_step.py only."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1903_12650_b200 import build as B  # noqa: E402

defs = [a for a in sys.argv[1:] if a.startswith("-D")]
tag = "".join(d[2:].split("=")[-1] for d in defs)
out = os.path.join(ROOT, "build", "trace" + tag)
os.makedirs(out, exist_ok=True)
nccl = B.nccl_root()
objs = []
for src in B.sources():
    obj = os.path.join(out, os.path.basename(src) + ".o")
    subprocess.check_call([B.NVCC, *B.ARCH, "-O3", "-std=c++17", "-lineinfo", "-DLARS_TRACE", *defs, "-Xcompiler", "-fPIC",
                           "-I", os.path.join(ROOT, "include"), "-I", B.CSRC, "-I", os.path.join(nccl, "include"),
                           "-c", src, "-o", obj])
    objs.append(obj)
lib = os.path.join(ROOT, "build", f"liblars_trace{tag}.so")
subprocess.check_call([B.NVCC, *B.ARCH, "-shared", "-cudart", "static", "-o", lib, *objs, "-L",
                       os.path.join(nccl, "lib"), "-l:libnccl.so.2", "-Xlinker", f"-rpath,{os.path.join(nccl, 'lib')}"])
print(lib)
