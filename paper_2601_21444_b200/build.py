"""Build recipe for libspava_b200.so (in-tree, sm_100a only).

    python -m paper_2601_21444_b200.build          # or __graft_entry__.build()

nvcc compiles every csrc/*.cu for `-gencode arch=compute_100a,code=sm_100a` with
-lineinfo (ncu source view) and links NCCL from the nvidia-nccl wheel torch ships
(rpath'd, so the GPU box resolves the same library).  No fast-math: the exact
scorer depends on IEEE double exp/div and explicit _rn intrinsics.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libspava_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    import importlib.util

    spec = importlib.util.find_spec("nvidia")
    cands = []
    if spec and spec.submodule_search_locations:
        for p in spec.submodule_search_locations:
            cands.append(os.path.join(p, "nccl"))
    for c in cands:
        if os.path.exists(os.path.join(c, "include", "nccl.h")):
            return os.path.join(c, "include"), os.path.join(c, "lib")
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))


def host_sources():
    """Host-only C++ (the seqpar:: mirror) is compiled by g++."""
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cpp")))


def needs_build():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + host_sources() + glob.glob(os.path.join(HERE, "csrc", "*.cuh")) + glob.glob(
        os.path.join(HERE, "csrc", "*.h")) + glob.glob(os.path.join(ROOT, "include", "*"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    inc, libdir = nccl_dirs()
    objs = []
    for src in host_sources():
        obj = os.path.join(HERE, "csrc", os.path.basename(src)[:-4] + ".o")
        r = subprocess.run(["g++", "-std=c++20", "-O2", "-fPIC", "-c", src, "-o", obj,
                            "-I", "/usr/local/cuda/include", "-I", os.path.join(ROOT, "include")],
                           capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("g++ failed:\n" + r.stdout + r.stderr)
        objs.append(obj)
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++20", "--expt-relaxed-constexpr",
           "-Xcompiler", "-fPIC,-O2", "-shared", "-I", inc, "-I", os.path.join(ROOT, "include"),
           *sources(), *objs, "-o", LIB + ".tmp", "-L", libdir, "-l:libnccl.so.2",
           "-Xlinker", f"-rpath,{libdir}"]
    if os.environ.get("SPAVA_DEV_VARIANTS") == "1":  # A/B kernel variants (dev build only)
        cmd.insert(1, "-DSPAVA_DEV_VARIANTS")
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + r.stdout + r.stderr)
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
