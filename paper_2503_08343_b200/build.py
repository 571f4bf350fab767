"""Builds libgmrf_b200.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import concurrent.futures
import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "_lib", "libgmrf_b200.so")
OBJ = os.path.join(HERE, "_obj")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
METIS = os.path.join(CUDA, "targets", "x86_64-linux", "lib", "libmetis_static.a")

NVCC_FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
              "-Xcompiler", "-fPIC", "-Wno-deprecated-gpu-targets"]
CXX_FLAGS = ["-O3", "-std=c++17", "-fPIC", "-march=x86-64-v3", f"-I{CUDA}/include"]


def _run(cmd):
    subprocess.run(cmd, check=True)


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    headers = glob.glob(os.path.join(CSRC, "*.hpp")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(HERE, "..", "include", "gmrf_b200.h")]
    objs, jobs = [], []
    for src in sorted(glob.glob(os.path.join(CSRC, "*.cpp"))):
        o = os.path.join(OBJ, os.path.basename(src) + ".o")
        if force or _stale(o, [src] + headers):
            jobs.append(["g++", *CXX_FLAGS, "-c", src, "-o", o])
        objs.append(o)
    for src in sorted(glob.glob(os.path.join(CSRC, "*.cu"))):
        if os.path.basename(src) == "kernels.cu":
            continue  # included by factor.cu (single device TU)
        o = os.path.join(OBJ, os.path.basename(src) + ".o")
        deps = [src, os.path.join(CSRC, "kernels.cu")] + headers
        if force or _stale(o, deps):
            jobs.append(["nvcc", *NVCC_FLAGS, "-c", src, "-o", o] +
                        (["-Xptxas", "-v"] if verbose else []))
        objs.append(o)
    # translation units compile in parallel (factor.cu dominates)
    with concurrent.futures.ThreadPoolExecutor(max_workers=max(1, min(len(jobs), 6))) as ex:
        for f in [ex.submit(_run, j) for j in jobs]:
            f.result()
    if force or _stale(LIB, objs):
        _run(["nvcc", "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", LIB, *objs,
              METIS, "-lcudart", "-lm", "-ldl"])
    return LIB


if __name__ == "__main__":
    import sys
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
