"""In-tree build of libbt_b200.so (CUDA sm_100a kernels + C++ host + C ABI).

nvcc compiles the .cu translation units for sm_100a only; the host .cpp
units are compiled by g++ without -march so the host-side setup arithmetic
(element matrices, stencil rows) keeps the reference's FMA-free rounding.
Run: python -m paper_2308_01792_b200.build  (or __graft_entry__.build()).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "libbt_b200.so")
OBJ = os.path.join(PKG, "build")

CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
            "-Xptxas", "-v"]
PER_FILE = {}  # per translation unit extra flags
CXX = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
CXX_FLAGS = ["-O2", "-std=c++17", "-fPIC", "-fno-fast-math", "-ffp-contract=off",
             f"-I{CUDA_HOME}/include"]

CU_SOURCES = ["bt_kernels.cu", "bt_stencil.cu", "bt_prism.cu", "bt_ew.cu", "bt_interface.cu", "bt_n1e1.cu", "bt_xchg.cu"]
CXX_SOURCES = ["bt_host.cpp", "bt_solvers.cpp", "bt_comm.cpp"]


def _deps(src=None):
    """A translation unit depends on itself and on every header."""
    hdrs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".hpp", ".h"))]
    return hdrs + [os.path.join(ROOT, "include", "blocktet_b200.h")] + (
        [os.path.join(CSRC, src)] if src else [])


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources if os.path.exists(s))


def _run(cmd, log):
    r = subprocess.run(cmd, capture_output=True, text=True)
    log.write(" ".join(cmd) + "\n" + r.stdout + r.stderr + "\n")
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build failed: {' '.join(cmd[:3])} ...")


def build(force: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    objs, jobs = [], []
    for src in CU_SOURCES:
        o = os.path.join(OBJ, src + ".o")
        if force or _stale(o, _deps(src)):
            jobs.append([NVCC, *ARCH, *CU_FLAGS, *PER_FILE.get(src, []), "-c", os.path.join(CSRC, src), "-o", o])
        objs.append(o)
    for src in CXX_SOURCES:
        o = os.path.join(OBJ, src + ".o")
        if force or _stale(o, _deps(src)):
            jobs.append([CXX, *CXX_FLAGS, "-c", os.path.join(CSRC, src), "-o", o])
        objs.append(o)
    with open(os.path.join(OBJ, "build.log"), "w") as log:
        # translation units compile in parallel (the logs are written in order)
        import concurrent.futures as cf
        import io
        logs = [io.StringIO() for _ in jobs]
        with cf.ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
            futs = [ex.submit(_run, cmd, lg) for cmd, lg in zip(jobs, logs)]
            errors = [f.exception() for f in futs]
        for lg in logs:
            log.write(lg.getvalue())
        for e in errors:
            if e is not None:
                raise e
        if force or _stale(OUT, objs):
            _run([NVCC, *ARCH, "-shared", "-o", OUT, *objs, "-lcudart_static", "-lrt", "-lpthread", "-ldl"], log)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
    if shutil.which("cuobjdump"):
        pass
