"""Builds libgrafem_b200.so in-tree (paper_2103_14870_b200/_lib/) for sm_100a.

nvcc compiles the CUDA translation units (-gencode arch=compute_100a,code=sm_100a -lineinfo); the
damage and per-node kernels are built with -fmad=false (bit-exact contract with the oracle), the
assembly and CG kernels with FMA. Host setup code is compiled with -ffp-contract=off.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "_lib")
OBJ = os.path.join(OUT, "obj")
LIB = os.path.join(OUT, "libgrafem_b200.so")
INC = os.path.join(os.path.dirname(HERE), "include")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_SOURCES = {  # file -> extra flags
    "damage.cu": ["-fmad=false"],
    "misc.cu": ["-fmad=false"],
    "assemble.cu": [],
    "cg.cu": [],
    "cg_sell.cu": [],
    "cg_onchip.cu": [],
    "sim.cu": [],
    "probe.cu": [],
    "metrics.cu": [],
}
CPP_SOURCES = ["host_mesh.cpp", "host_viz.cpp", "capi.cpp"]


def _nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _host_cxx():
    # the distro g++ links libstdc++/libgomp dynamically (the /opt/gcc wrapper in this image does not)
    for c in ("/usr/bin/x86_64-linux-gnu-g++-13", "/usr/bin/aarch64-linux-gnu-g++-13", "/usr/bin/g++", shutil.which("g++")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("no host C++ compiler")


def _cuda_home(nvcc):
    return os.path.dirname(os.path.dirname(os.path.realpath(nvcc)))


def _run(cmd):
    r = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed:\n" + " ".join(cmd) + "\n" + r.stdout)
    return r.stdout


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, ptxas_info: bool = False) -> str:
    nvcc = _nvcc()
    cxx = _host_cxx()
    os.makedirs(OBJ, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".hpp"))]
    headers.append(os.path.join(INC, "grafem_b200.h"))
    common_host = ["-O3", "-std=c++17", "-fPIC", "-fopenmp", "-ffp-contract=off", "-fno-fast-math"]
    jobs = []
    objs = []
    for f, extra in CU_SOURCES.items():
        src = os.path.join(CSRC, f)
        obj = os.path.join(OBJ, f + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + headers):
            cmd = [nvcc, "-c", src, "-o", obj, "-O3", "-std=c++17", "-lineinfo", *ARCH, "-ccbin", cxx,
                   "-Xcompiler", ",".join(common_host), "-I", INC, *extra]
            if ptxas_info:
                cmd += ["-Xptxas", "-v"]
            jobs.append(cmd)
    cuda_inc = os.path.join(_cuda_home(nvcc), "include")
    for f in CPP_SOURCES:
        src = os.path.join(CSRC, f)
        obj = os.path.join(OBJ, f + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + headers):
            jobs.append([cxx, "-c", src, "-o", obj, *common_host, "-I", INC, "-I", cuda_inc])
    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(8, len(jobs))) as ex:
            for out in ex.map(_run, jobs):
                if verbose and out:
                    print(out, file=sys.stderr)
    if force or jobs or _stale(LIB, objs):
        _run([nvcc, "-shared", "-o", LIB, *objs, *ARCH, "-ccbin", cxx, "-Xcompiler", "-fopenmp", "-lgomp"])
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True, ptxas_info="--ptxas" in sys.argv)
    print(LIB)
