"""Builds the C-ABI shared library libnbldpc.so for sm_100a with nvcc (in-tree)."""

from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.environ.get("NBLDPC_LIB", os.path.join(LIBDIR, "libnbldpc.so"))  # override: tuning builds
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh")) +
                  glob.glob(os.path.join(CSRC, "*.h")) + [os.path.join(ROOT, "include", "nbldpc.h")])


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every csrc/*.cu translation unit to an object in parallel (the kernel families live in
    separate units, csrc/k_*.cu), then link libnbldpc.so."""
    newest = max(os.path.getmtime(s) for s in sources())
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= newest:
        return LIB
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    tag = f"tmp{os.getpid()}"
    objdir = os.path.join(os.path.dirname(LIB), f"obj.{tag}")
    os.makedirs(objdir, exist_ok=True)
    defs = os.environ.get("NBLDPC_DEFS", "").split()  # e.g. "-DNB_CLUSTER_MINB=2" (tuning builds)
    common = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", *defs,
              "-Xptxas", "-v" if verbose else "-O3"]
    units = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    objs = [os.path.join(objdir, os.path.basename(u)[:-3] + ".o") for u in units]

    def compile_unit(i):
        return subprocess.run([*common, "-c", units[i], "-o", objs[i]], capture_output=True, text=True)

    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(max_workers=min(len(units), os.cpu_count() or 1)) as ex:
        results = list(ex.map(compile_unit, range(len(units))))
    failed = [(u, r) for u, r in zip(units, results) if r.returncode != 0]
    if verbose:
        for r in results:
            sys.stderr.write(r.stderr)
    import shutil

    try:
        if failed:
            for u, r in failed:
                sys.stderr.write(f"--- {u}\n" + r.stdout + r.stderr)
            raise RuntimeError("nvcc failed building libnbldpc.so")
        tmp = LIB + "." + tag
        res = subprocess.run([NVCC, *ARCH, "-shared", "-o", tmp, *objs], capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError("nvcc failed linking libnbldpc.so")
        os.replace(tmp, LIB)
    finally:
        shutil.rmtree(objdir, ignore_errors=True)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
