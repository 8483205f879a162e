"""Build librdr.so in-tree: nvcc for the sm_100a kernels, g++ (OpenMP) for the
host setup and the C ABI. Usage: python -m paper_2506_17406_b200.build"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "librdr.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
HOST_FLAGS = ["-O3", "-std=c++17", "-fPIC", "-fopenmp", "-march=x86-64-v3", "-Wall", "-Wno-unused-function", "-Wno-array-bounds"]


def _run(cmd):
    print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def build(verbose_ptxas: bool = False) -> str:
    bdir = os.path.join(HERE, "_build")
    os.makedirs(bdir, exist_ok=True)
    objs = []
    kflags = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", *ARCH]
    if verbose_ptxas:
        kflags += ["-Xptxas", "-v"]
    for cu in ("kernels.cu", "patch_setup.cu"):
        o = os.path.join(bdir, cu + ".o")
        _run([NVCC, *kflags, "-c", os.path.join(CSRC, cu), "-o", o])
        objs.append(o)
    for cpp in ("refelem.cpp", "setup.cpp", "dense.cpp", "rdr_abi.cpp"):
        o = os.path.join(bdir, cpp + ".o")
        _run(["g++", *HOST_FLAGS, "-I", os.path.join(CUDA, "include"), "-c", os.path.join(CSRC, cpp), "-o", o])
        objs.append(o)
    _run(["g++", "-shared", "-fopenmp", "-o", OUT, *objs, "-L", os.path.join(CUDA, "lib64"), "-lcudart",
          f"-Wl,-rpath,{os.path.join(CUDA, 'lib64')}"])
    return OUT


if __name__ == "__main__":
    build(verbose_ptxas="-v" in sys.argv)
