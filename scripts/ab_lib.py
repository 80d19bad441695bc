#!/usr/bin/env python
"""A/B builds: recompile one translation unit with extra nvcc flags (e.g. -DNAME)
and link it with the other objects of the in-tree build into
paper_1602_08393_b200/libwmh_<tag>.so, loaded by scripts via WMH_LIB_AB.

    python scripts/ab_lib.py <tag> <unit.cu> [-DFLAG ...]
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1602_08393_b200 import build as b  # noqa: E402


def main(tag, unit, *flags):
    b.build()
    objdir = os.path.join(b.PKG, "build")
    src = os.path.join(b.CSRC, unit)
    obj = os.path.join(objdir, f"ab_{tag}_{unit}.o")
    subprocess.run(["nvcc", *b.NVCC_FLAGS, *flags, "-I", b.INCLUDE, "-I", b.CSRC, "-c", src, "-o", obj], check=True,
                   capture_output=True)
    objs = [os.path.join(objdir, os.path.basename(s) + ".o") for s in b.sources()]
    objs = [obj if os.path.basename(o) == unit + ".o" else o for o in objs]
    so = os.path.join(b.PKG, f"libwmh_{tag}.so")
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC", "-cudart",
                    "shared", "-Xlinker", "-rpath=/usr/local/cuda/lib64", "-o", so, *objs], check=True)
    os.remove(obj)
    print(so)


if __name__ == "__main__":
    main(*sys.argv[1:])
