"""Build libhercules_rec.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

The library is plain C ABI (include/rec.h); Python reaches it through ctypes
(paper_2203_07424_b200/binding.py).  Object files are cached under build/ keyed on
source mtimes; the .so is written next to this file so it travels with gpurun.
"""
from __future__ import annotations

import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libhercules_rec.so")
BUILD = os.path.join(ROOT, "build", "obj")

SOURCES = ["k_synth.cu", "k_sls.cu", "k_gemm.cu", "k_mlp.cu", "k_interact.cu", "model.cu", "pipe.cu", "dist.cu",
           "serve.cpp"]
HEADERS = ["common.cuh", "sm100.cuh", "kernels.h", "model.h", "synth.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dir() -> str:
    site = sysconfig.get_paths()["purelib"]
    d = os.path.join(site, "nvidia", "nccl")
    if not os.path.isdir(d):
        raise RuntimeError(f"NCCL headers/library not found under {d}")
    return d


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def build(verbose: bool = False, force: bool = False, defines=(), out: str = OUT,
          objdir: str = BUILD) -> str:
    """Compile every source for sm_100a and link `out`.  `defines` (e.g. REC_MBAR_SPIN) go to
    every translation unit; use a separate `objdir` for variant builds."""
    BUILD_ = objdir
    os.makedirs(BUILD_, exist_ok=True)
    dflags = [f"-D{d}" for d in defines]
    nccl = _nccl_dir()
    inc = ["-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", os.path.join(nccl, "include")]
    hdr_mtime = max(os.path.getmtime(os.path.join(CSRC, h)) for h in HEADERS)
    hdr_mtime = max(hdr_mtime, os.path.getmtime(os.path.join(ROOT, "include", "rec.h")))
    objs = []
    for src in SOURCES:
        sp = os.path.join(CSRC, src)
        op = os.path.join(BUILD_, src + ".o")
        objs.append(op)
        if not force and os.path.exists(op) and os.path.getmtime(op) > max(os.path.getmtime(sp), hdr_mtime):
            continue
        if src.endswith(".cu"):
            cmd = [_nvcc(), *ARCH, "-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC",
                   "-Xcompiler", "-ffp-contract=off", "--expt-relaxed-constexpr", *dflags, *inc,
                   "-c", sp, "-o", op]
        else:
            cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-pthread", *dflags,
                   "-I", "/usr/local/cuda/include", *inc, "-c", sp, "-o", op]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
    link = [_nvcc(), *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", out, *objs,
            "-L", os.path.join(nccl, "lib"), "-l:libnccl.so.2",
            "-Xlinker", "-rpath=" + os.path.join(nccl, "lib"), "-lpthread"]
    if force or not os.path.exists(out) or os.path.getmtime(out) < max(os.path.getmtime(o) for o in objs):
        if verbose:
            print(" ".join(link), file=sys.stderr)
        subprocess.run(link, check=True)
    return out


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv))
