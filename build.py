"""Build the in-tree native libraries.

  paper_1812_06856_b200/liblfdg.so   the product: sm_100a CUDA kernels + C-ABI (include/lfdg.h)
                                      + host C++ (scene generator), nvcc -gencode arch=compute_100a,code=sm_100a
  oracle/_build/liblfdoracle.so       test infrastructure: the plain-C restatement (oracle/lfd_oracle.c)
  oracle/_ref/liblfdref.so            test infrastructure: the unmodified reference headers + shims
                                      (only when /root/reference is present, i.e. not on the GPU box)

FP contract: --fmad=false and -ffp-contract=off everywhere on the parity path.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
PKG = os.path.join(ROOT, "paper_1812_06856_b200")
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "liblfdg.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "--fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-O3",
    "-shared",
]


def _stale(target: str, sources) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def build_product(force: bool = False, verbose: bool = False) -> str:
    """One nvcc per translation unit (in parallel, objects under build/), then one link."""
    from concurrent.futures import ThreadPoolExecutor

    sources = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))
    headers = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + [
        os.path.join(ROOT, "include", "lfdg.h")]
    odir = os.path.join(ROOT, "build")
    os.makedirs(odir, exist_ok=True)
    compile_flags = [f for f in NVCC_FLAGS if f != "-shared"]

    def obj(src):
        o = os.path.join(odir, os.path.basename(src) + ".o")
        if force or _stale(o, [src] + headers):
            cmd = ["nvcc", *compile_flags, "-c", src, "-o", o]
            if verbose:
                print(" ".join(cmd), flush=True)
            subprocess.run(cmd, check=True, cwd=ROOT)
        return o

    with ThreadPoolExecutor(max_workers=max(1, min(len(sources), os.cpu_count() or 1))) as ex:
        objs = list(ex.map(obj, sources))
    if force or _stale(LIB, objs):
        cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", *objs, "-o", LIB]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True, cwd=ROOT)
    return LIB


def build_oracle(verbose: bool = False) -> None:
    odir = os.path.join(ROOT, "oracle")
    if os.path.exists(os.path.join(odir, "lfd_oracle.c")):
        subprocess.run(["make", "-s", "_build/liblfdoracle.so"], cwd=odir, check=True)
    if os.path.isdir("/root/reference/proj/include"):
        subprocess.run(["make", "-s", "ref"], cwd=odir, check=True)
        subprocess.run(["make", "-s", "gpu-dropin-tests"], cwd=odir, check=True)


def main() -> None:
    force = "--force" in sys.argv
    build_product(force=force, verbose=True)
    build_oracle(verbose=True)


if __name__ == "__main__":
    main()
