"""Build the in-tree CUDA library libpbicgstab.so for sm_100a with nvcc.

nvcc cross-compiles without a GPU, so this runs on the CPU build box too.
"""
from __future__ import annotations

import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libpbicgstab.so")
ROOT = os.path.dirname(HERE)

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",            # no FMA contraction anywhere (reading A4)
    "-Xcompiler", "-ffp-contract=off",  # host-side constants (block inverses, bounds) too
    "-Xcompiler", "-fPIC",
    "-diag-suppress", "177",
]

# translation units: the host driver (+ Jacobi kernels) and the block-Jacobi tile
# instances, one object per block size, compiled in parallel and linked into one .so
UNITS = [("pbicgstab.cu", []), ("tile_bj.cu", ["-DPBICG_BJ_B=2"]),
         ("tile_bj.cu", ["-DPBICG_BJ_B=4"]), ("tile_bj.cu", ["-DPBICG_BJ_B=8"]),
         ("tile_seg.cu", []), ("tile_jac.cu", ["-DPBICG_VEC=1"]),
         ("tile_jac.cu", ["-DPBICG_VEC=0"])]


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                  + glob.glob(os.path.join(CSRC, "*.h"))
                  + [os.path.join(ROOT, "include", "pbicgstab.h")])


def nvcc() -> str:
    for c in ("/usr/local/cuda/bin/nvcc", "nvcc"):
        if os.path.sep not in c or os.path.exists(c):
            return c
    return "nvcc"


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in sources())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    procs, objs = [], []
    for i, (src, defs) in enumerate(UNITS):
        obj = os.path.join(objdir, f"unit{i}.o")
        cmd = [nvcc(), *NVCC_FLAGS, *defs, "-c", "-o", obj, os.path.join(CSRC, src)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                                            text=True)))
        objs.append(obj)
    failed = []
    for cmd, p in procs:
        out, err = p.communicate()
        if p.returncode != 0:
            failed.append(f"{' '.join(cmd[-3:])}: {out}\n{err}")
        elif verbose:
            print(out, err)
    if failed:
        raise RuntimeError("nvcc failed:\n" + "\n".join(failed))
    link = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB, *objs]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc link failed ({r.returncode}):\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    build(force=True, verbose="-v" in __import__("sys").argv)
    print(LIB)
