"""In-tree build of libwmh.so (the CUDA path) for sm_100a with plain nvcc."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
# WMH_LIB=debug: a second library built with -DWMH_DEBUG, whose kernels check
# their shared/global indices with device-side asserts (WMH_DASSERT) -- the
# bounds checking used where compute-sanitizer is not available
DEBUG = os.environ.get("WMH_LIB") == "debug"
SO = os.path.join(PKG, "libwmh_debug.so" if DEBUG else "libwmh.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
    "-Xptxas", "-v",
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [os.path.join(INCLUDE, "wmh.h")]


def needs_build() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(p) > t for p in deps())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return SO
    # one builder at a time (torchrun starts one process per GPU): the others
    # wait on the lock and then find the library up to date
    import fcntl
    with open(os.path.join(PKG, ".build.lock"), "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        try:
            if not force and not needs_build():
                return SO
            return _build(verbose)
        finally:
            fcntl.flock(lk, fcntl.LOCK_UN)


def _build(verbose: bool) -> str:
    nvcc = os.environ.get("NVCC", "nvcc")
    objdir = os.path.join(PKG, "build_debug" if DEBUG else "build")
    os.makedirs(objdir, exist_ok=True)
    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [nvcc, *NVCC_FLAGS, *(["-DWMH_DEBUG"] if DEBUG else []), "-I", INCLUDE, "-I", CSRC, "-c", src, "-o", obj]
        return src, obj, subprocess.run(cmd, capture_output=True, text=True)

    # translation units compile in parallel (the two big template files dominate)
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=max(1, min(len(sources()), os.cpu_count() or 1))) as ex:
        results = list(ex.map(compile_one, sources()))
    objs = []
    log = []
    for src, obj, r in results:
        log.append(r.stdout + r.stderr)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        objs.append(obj)
    tmp = SO + f".tmp{os.getpid()}"
    # the shared CUDA runtime (the process's libcudart.so.12 -- torch's when torch is
    # loaded -- instead of a static copy inside libwmh.so); rpath for standalone use
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
           "-cudart", "shared", "-Xlinker", "-rpath=/usr/local/cuda/lib64", "-o", tmp, *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(tmp, SO)
    with open(os.path.join(objdir, "ptxas.log"), "w") as f:
        f.write("\n".join(log))
    if verbose:
        print("\n".join(log))
    return SO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
