"""In-tree build of librkb200.so (nvcc, sm_100a only).

    python -m paper_2309_05331_b200.build [--force]

Flags: -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo, -fmad=false (no FMA
contraction anywhere: the bitwise contract of DESIGN.md R-17), IEEE division/sqrt,
no flush-to-zero.  Links the NCCL shipped with the PyTorch wheel (same copy torch loads).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
import sysconfig

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(ROOT, "build", "rkb200")
LIB = os.path.join(PKG, "librkb200.so")
SOURCES = ["rk_runtime.cu", "rk_stencil.cu", "rk_pointwise.cu", "rk_algebra.cu", "rk_smallgrid.cu", "rk_fused.cu",
           "rk_fused2.cu", "rk_pair.cu"]
HEADERS = ["rk_kernels.cuh", "rk_device.cuh", "rk_tableau.h", "rk_stage_spec.h", "rk_ddmath.cuh"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-fmad=false", "-prec-div=true",
                     "-prec-sqrt=true", "-ftz=false", "--expt-relaxed-constexpr",
                     "-Xcompiler", "-fPIC,-O2,-ffp-contract=off", "-Xptxas", "-v"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def nccl_dir() -> str:
    cands = [os.path.join(p, "nvidia", "nccl") for p in sys.path if p] + \
            [os.path.join(sysconfig.get_paths()["purelib"], "nvidia", "nccl")]
    for c in cands:
        if os.path.exists(os.path.join(c, "include", "nccl.h")):
            return c
    raise RuntimeError("NCCL headers (nvidia/nccl in site-packages) not found")


def _stale(out: str, deps: list[str]) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    nd = nccl_dir()
    inc = ["-I", INCLUDE, "-I", CSRC, "-I", os.path.join(nd, "include")]
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(INCLUDE, "rk_b200.h")]
    objs, jobs = [], []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _stale(o, [s] + hdrs + [os.path.abspath(__file__)]):
            jobs.append([nvcc(), *NVCC_FLAGS, *os.environ.get("RKB_NVCC_EXTRA", "").split(), *inc, "-c", s, "-o", o])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        return r.stderr

    with cf.ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        for log in ex.map(run, jobs):
            if verbose:
                print(log)
    if force or jobs or _stale(LIB, objs):
        tmp = LIB + f".tmp{os.getpid()}"
        run([nvcc(), *ARCH, "-shared", "-o", tmp, *objs, "-L", os.path.join(nd, "lib"),
             "-l:libnccl.so.2", "-Xlinker", "-rpath=" + os.path.join(nd, "lib")])
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
