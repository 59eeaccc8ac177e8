"""Build libcc.so (the CUDA path) in-tree with nvcc for sm_100a.

`python -m paper_2604_18801_b200.build` or `__graft_entry__.build()`.  nvcc cross-compiles
without a GPU.  Flags: -O3, -lineinfo (ncu source view), -fmad=false (no FMA contraction
anywhere: the pinned fp32 expressions of DESIGN.md R4/R9/R14 must round every operation).
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
LIB = os.path.join(HERE, "libcc.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _nccl_dir():
    import nvidia.nccl  # torch's bundled NCCL 2.28 (headers + libnccl.so.2)
    return os.path.dirname(list(nvidia.nccl.__path__)[0] + "/")


NCCL = _nccl_dir()
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-fmad=false", "-Xcompiler", "-fPIC", "-Xptxas", "-warn-spills",
         f"-I{INCLUDE}", f"-I{os.path.join(NCCL, 'include')}"]
LDFLAGS = [f"-L{os.path.join(NCCL, 'lib')}", "-l:libnccl.so.2", "-Xlinker", f"-rpath={os.path.join(NCCL, 'lib')}"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(INCLUDE, "*.h"))
    if not force and not _stale(LIB, deps):
        return LIB
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
        if force or _stale(obj, [src] + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(INCLUDE, "*.h"))):
            cmd = [NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj]
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            try:
                subprocess.check_call(cmd)
            except subprocess.CalledProcessError:
                for f in (obj, LIB):  # never leave a stale library behind a failed build
                    if os.path.exists(f):
                        os.remove(f)
                raise
        objs.append(obj)
    tmp = LIB + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, *ARCH, "-shared", "-o", tmp, *objs, *LDFLAGS])
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
