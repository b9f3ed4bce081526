"""Build libvlp.so in-tree: nvcc for sm_100a (kernels + device API), g++ for the host C++.

    python -m paper_2506_12761_b200.build [--force]
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
# VLP_BUILD_VARIANT=name (dev tools only): extra -D flags from VLP_BUILD_DEFS, objects and library under other names
VARIANT = os.environ.get("VLP_BUILD_VARIANT", "")
DEFS = os.environ.get("VLP_BUILD_DEFS", "").split() if VARIANT else []
BUILD = os.path.join(HERE, "_build" + (f"_{VARIANT}" if VARIANT else ""))
LIB = os.path.join(HERE, f"libvlp_{VARIANT}.so" if VARIANT else "libvlp.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU = ["kernels.cu", "kernels_fft.cu", "kernels_ks.cu", "api.cu"]
CXX = ["host.cpp", "sched.cpp"]
HDR = ["vlp_internal.h", "kernels.cuh", "devcommon.cuh", os.path.join("..", "..", "include", "vlp.h")]


def _newer(src_list, target):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(os.path.join(CSRC, s)) > t for s in src_list)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    objs = []
    for f in CU:
        o = os.path.join(BUILD, f + ".o")
        if force or _newer([f] + HDR, o):
            cmd = [NVCC, *ARCH, *DEFS, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
                   "-c", os.path.join(CSRC, f), "-o", o]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed on {f}")
            with open(os.path.join(BUILD, f + ".ptxas.txt"), "w") as fh:
                fh.write(r.stderr)
            if verbose:
                sys.stderr.write(r.stderr)
        objs.append(o)
    for f in CXX:
        o = os.path.join(BUILD, f + ".o")
        if force or _newer([f] + HDR, o):
            cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-fno-fast-math", "-pthread",
                   "-I/usr/local/cuda/include", "-c", os.path.join(CSRC, f), "-o", o]
            subprocess.check_call(cmd)
        objs.append(o)
    if force or not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        subprocess.check_call([NVCC, *ARCH, "-shared", "-o", LIB + ".tmp", *objs, "-Xcompiler", "-pthread",
                               "-Xlinker", "-rpath=/usr/local/cuda/lib64"])
        os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
