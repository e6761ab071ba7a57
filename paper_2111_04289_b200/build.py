"""Build the in-tree shared libraries for sm_100a (nvcc; no GPU needed to compile).

  paper_2111_04289_b200/liblmstream.so   the product (C ABI in include/lmstream.h)
  lmsgen/liblmsgen.so                    the CUDA input generator (test / bench input only)

Usage: python paper_2111_04289_b200/build.py [--force]   (or __graft_entry__.build())
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "-cudart", "static",
          "--expt-relaxed-constexpr", "-Xptxas", "-v"]

LIB = os.path.join(PKG, "liblmstream.so")
GEN_LIB = os.path.join(ROOT, "lmsgen", "liblmsgen.so")


def _sources(pattern_dir, exts=(".cu", ".cpp")):
    out = []
    for e in exts:
        out += glob.glob(os.path.join(pattern_dir, "*" + e))
    return sorted(out)


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _nvcc(out, srcs, extra=(), log=None):
    cmd = [NVCC, *ARCH, *COMMON, "-shared", "-o", out + ".tmp", *srcs, *extra]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if log is not None:
        with open(log, "w") as fh:
            fh.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"nvcc failed building {out}")
    os.replace(out + ".tmp", out)


def build(force: bool = False, verbose: bool = False) -> None:
    csrc = os.path.join(PKG, "csrc")
    srcs = _sources(csrc)
    deps = srcs + glob.glob(os.path.join(csrc, "*.h")) + glob.glob(os.path.join(csrc, "*.cuh")) + \
        [os.path.join(ROOT, "include", "lmstream.h")]
    if force or _stale(LIB, deps):
        _nvcc(LIB, srcs, ["-I", os.path.join(ROOT, "include")], log=os.path.join(PKG, "build_ptxas.log"))
        if verbose:
            print("built", LIB)
    gsrc = [os.path.join(ROOT, "lmsgen", "gen.cu")]
    if os.path.exists(gsrc[0]) and (force or _stale(GEN_LIB, gsrc)):
        _nvcc(GEN_LIB, gsrc)
        if verbose:
            print("built", GEN_LIB)


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
