"""Build libkafmm_<name>.so with extra nvcc -D flags (A/B tuning of compile-time
knobs; select at run time with KAFMM_LIB=<path>).

    python scripts/build_variant.py minb6 -DKF_DMMA_MINB1=6 -DKF_DMMA_MINB3=4
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2010_15155_b200 import build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(B.HERE, f"libkafmm_{name}.so")
bdir = os.path.join(B.BUILD, name)
os.makedirs(bdir, exist_ok=True)
objs = []
for src in B.SOURCES:
    obj = os.path.join(bdir, src.replace(".cu", ".o"))
    subprocess.run([B.nvcc(), *B.ARCH, *B.FLAGS, *defs, "-c", os.path.join(B.CSRC, src), "-o", obj], check=True)
    objs.append(obj)
subprocess.run([B.nvcc(), *B.ARCH, "-shared", "-o", out, *objs, "-lcublas", "-lcusolver", "-lcufft", "-lcudart", "-ldl"],
               check=True)
print(out)
