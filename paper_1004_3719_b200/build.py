"""Build libffspmv.so in-tree for sm_100a.

    python -m paper_1004_3719_b200.build [--force]

CUDA sources are compiled with ``nvcc -gencode arch=compute_100a,code=sm_100a
-lineinfo -O3``; host sources with g++; everything is linked into
``paper_1004_3719_b200/libffspmv.so`` with the CUDA runtime linked
statically.  ptxas register/spill reports go to ``build/ptxas.log``.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", "ffspmv")
LIB = os.path.join(PKG, "libffspmv.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")

CU_SOURCES = ["seq.cu", "block.cu", "block16.cu", "block16w.cu", "block8.cu", "kernels.cu", "panel.cu", "runs.cu"]
CPP_SOURCES = ["abi.cpp", "builder.cpp", "panel_build.cpp", "runs_build.cpp", "comm.cpp"]
HEADERS = ["internal.hpp", "device.cuh", "block.cuh", "seq_mma.cuh", "comm.hpp", "l2window.hpp"]
GENCODE = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _newer(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return r.stdout + r.stderr


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "ffspmv.h")]
    jobs = []
    objs = []
    for s in CU_SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(BUILD, s + ".o")
        objs.append(obj)
        if force or _newer(obj, [src] + hdrs):
            jobs.append([NVCC, "-std=c++17", "-O3", "-lineinfo", *GENCODE, "-Xptxas", "-v",
                         "-Xcompiler", "-fPIC,-fvisibility=hidden", "-I", CSRC,
                         "-c", src, "-o", obj])
    for s in CPP_SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(BUILD, s + ".o")
        objs.append(obj)
        if force or _newer(obj, [src] + hdrs):
            jobs.append(["g++", "-std=c++17", "-O3", "-fPIC", "-fvisibility=hidden", "-Wall",
                         "-I", os.path.join(CUDA, "include"), "-I", CSRC, "-c", src, "-o", obj])
    logs = []
    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(8, len(jobs))) as ex:
            for job, out in zip(jobs, ex.map(_run, jobs)):
                logs.append(out)
                with open(job[job.index("-o") + 1] + ".log", "w") as f:   # per-object ptxas report
                    f.write(out)
    if force or jobs or _newer(LIB, objs):
        tmp = LIB + f".tmp{os.getpid()}"
        _run([NVCC, "-shared", *GENCODE, "-cudart", "static", "-o", tmp, *objs,
              "-Xlinker", "--exclude-libs,ALL", "-ldl"])
        os.replace(tmp, LIB)
    if verbose:
        print("\n".join(logs))
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
