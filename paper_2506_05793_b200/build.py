"""Build libfastilu_b200.so in-tree (nvcc for sm_100a + g++ for the host setup).

    python -m paper_2506_05793_b200.build [--force] [--verbose]

The library is written to paper_2506_05793_b200/lib/libfastilu_b200.so (git-ignored; it travels
to the GPU box with the gpurun snapshot).  The CUDA runtime is linked statically.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "lib", "libfastilu_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_SRCS = ["kernels.cu", "bsr.cu", "fastilu.cu"]
CXX_SRCS = ["symbolic.cpp", "comm.cpp", "classes.cpp", "tsell.cpp", "jit.cpp", "blocks.cpp"]
HDRS = ["host.h", "device.h", "comm.h", "tsell.h", "jit.h", "blocks.h"]


def _sources():
    return [os.path.join(CSRC, s) for s in CU_SRCS + CXX_SRCS + HDRS] + \
        [os.path.join(ROOT, "include", "fastilu.h"), os.path.abspath(__file__)]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale(LIB, _sources()):
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    inc = ["-I" + os.path.join(ROOT, "include"), "-I" + CSRC, "-I/usr/local/cuda/include"]
    jobs = []
    objs = []
    for s in CU_SRCS:
        o = os.path.join(OBJ, s + ".o")
        objs.append(o)
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
               "-Xptxas", "-v" if verbose else "-O3", "-c", os.path.join(CSRC, s), "-o", o, *inc]
        jobs.append(cmd)
    for s in CXX_SRCS:
        o = os.path.join(OBJ, s + ".o")
        objs.append(o)
        cmd = ["g++", "-O3", "-std=c++17", "-fPIC", "-pthread", "-c", os.path.join(CSRC, s),
               "-o", o, *inc]
        jobs.append(cmd)
    procs = [(c, subprocess.Popen(c, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
             for c in jobs]
    failed = False
    for c, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            failed = True
            sys.stderr.write(" ".join(c) + "\n" + out + "\n")
        elif verbose and out:
            sys.stderr.write(out)
    if failed:
        raise RuntimeError("libfastilu_b200 build failed")
    tmp = LIB + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lpthread", "-ldl"])
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv))
