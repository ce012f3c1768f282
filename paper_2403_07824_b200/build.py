"""In-tree build of the CUDA library ``paper_2403_07824_b200/libvqpc.so``.

nvcc cross-compiles for sm_100a only (``-gencode arch=compute_100a,code=sm_100a``)
with ``-lineinfo`` so ncu's source page maps to the kernels. Host code is
compiled with ``-ffp-contract=off`` (no FMA contraction on the host side, like
the reference's Release build without ``-march``).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.environ.get("VQPC_LIB", os.path.join(HERE, "libvqpc.so"))
SOURCES = ["vqpc.cu", "host_quantizer.cu", "klbasis.cu"]
HEADERS = ["amg_setup.cuh", "pcgamg2d.cuh", "common.cuh", "realise.cuh", "assign.cuh", "bucket.cuh", "factor.cuh", "pcg1d.cuh", "pcg1d_exact.cuh", "pcg2d.cuh", "pcgchol2d.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
EXTRA = os.environ.get("VQPC_NVCC_FLAGS", "").split()
FLAGS = [*EXTRA, "-O3", "-lineinfo", "-std=c++20", "-Xcompiler", "-fPIC,-ffp-contract=off", "-Xptxas", "-v",
         "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"), "-I", CSRC]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "vqpc.h"), __file__]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    objdir = os.path.join(HERE, "build" + ("_" + os.path.basename(LIB).replace(".so", "") if "VQPC_LIB" in os.environ else ""))
    os.makedirs(objdir, exist_ok=True)
    objs = []
    for s in SOURCES:
        o = os.path.join(objdir, s.replace(".cu", ".o"))
        cmd = [NVCC, *ARCH, *FLAGS, "-c", os.path.join(CSRC, s), "-o", o]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {s}")
        with open(os.path.join(objdir, s + ".ptxas.log"), "w") as f:
            f.write(r.stderr)
        if verbose:
            sys.stderr.write(r.stderr)
        objs.append(o)
    cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lpthread", "-lcublas"]
    subprocess.check_call(cmd)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
