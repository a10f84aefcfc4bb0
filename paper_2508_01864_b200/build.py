"""Build libgpmatern.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

    python -m paper_2508_01864_b200.build        # or __graft_entry__.build()
"""
from __future__ import annotations

import os
import subprocess
import sys
import concurrent.futures as cf

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
# experiment builds: GPM_LIB_SUFFIX=_x GPM_EXTRA_FLAGS="-DFOO=1" -> libgpmatern_x.so (load it with
# GPM_LIB=<path>); the product build uses neither
SUFFIX = os.environ.get("GPM_LIB_SUFFIX", "")
LIB = os.path.join(HERE, f"libgpmatern{SUFFIX}.so")
OBJDIR = os.path.join(HERE, "build" + SUFFIX)
SOURCES = ["api.cu", "setup.cu", "apply.cu", "apply_d1.cu", "apply_d1_big.cu", "apply_level.cu",
           "apply_level_p1.cu", "apply_level_p2.cu", "apply_level_p3.cu", "solve.cu", "lml.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr",
         "-Xptxas", "-v" if os.environ.get("GPM_PTXAS_V") else "-O3",
         *os.environ.get("GPM_EXTRA_FLAGS", "").split()]


def _newer(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    hs.append(os.path.join(CSRC, "apply_level.cu"))   # included by apply_level_p{1,2,3}.cu
    hs.append(os.path.join(os.path.dirname(HERE), "include", "gpmatern.h"))
    return hs


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJDIR, exist_ok=True)
    hdrs = _headers()
    jobs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJDIR, src.replace(".cu", ".o"))
        if force or _newer(o, [s] + hdrs):
            jobs.append((s, o))

    def run(job):
        s, o = job
        cmd = [NVCC, *FLAGS, "-c", s, "-o", o]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {s}:\n{r.stdout}\n{r.stderr}")
        return r.stderr

    with cf.ThreadPoolExecutor(max_workers=min(len(jobs) or 1, os.cpu_count() or 4)) as ex:
        for log in ex.map(run, jobs):
            if verbose and log:
                print(log, file=sys.stderr)
    objs = [os.path.join(OBJDIR, s.replace(".cu", ".o")) for s in SOURCES]
    if force or jobs or _newer(LIB, objs):
        tmp = LIB + f".tmp{os.getpid()}"
        cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", tmp, *objs,
               "-lcudart", "-lcublas"]
        subprocess.check_call(cmd)
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
