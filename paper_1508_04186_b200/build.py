"""Build libdqn.so (the C-ABI product library) in-tree for sm_100a.

nvcc cross-compiles without a GPU; the .so travels to the GPU box with the repo
snapshot. NCCL is linked from the torch wheel (nvidia/nccl) so one process never
loads two different libnccl builds.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libdqn.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dir() -> str:
    import nvidia.nccl  # the wheel torch links against

    return list(nvidia.nccl.__path__)[0]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) +
                  glob.glob(os.path.join(ROOT, "include", "*.h")))


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(f) <= t for f in sources() + headers() + [__file__])


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    nd = nccl_dir()
    objdir = os.path.join(PKG, "build")
    os.makedirs(objdir, exist_ok=True)
    common = ["nvcc", *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v" if verbose else "-O3",
              "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", os.path.join(nd, "include")]
    objs = []
    procs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        procs.append(subprocess.Popen(common + ["-c", src, "-o", obj]))
    rc = [p.wait() for p in procs]
    if any(rc):
        raise RuntimeError("nvcc failed")
    link = ["nvcc", *ARCH, "-shared", "-o", LIB + ".tmp", *objs, "-L", os.path.join(nd, "lib"), "-l:libnccl.so.2",
            "-Xlinker", "-rpath," + os.path.join(nd, "lib")]
    subprocess.check_call(link)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
