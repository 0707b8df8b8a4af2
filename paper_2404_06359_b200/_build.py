"""Build libmc.so in-tree: host encoder (g++) + sm_100a decode kernels (nvcc).

    python -m paper_2404_06359_b200._build
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libmc.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
SOURCES = [os.path.join(CSRC, "encode.cpp"), os.path.join(CSRC, "decode.cu"),
           os.path.join(ROOT, "include", "mc.h")]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in SOURCES)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    bdir = os.path.join(PKG, "build")
    os.makedirs(bdir, exist_ok=True)
    enc_o = os.path.join(bdir, "encode.o")
    dec_o = os.path.join(bdir, "decode.o")
    cmds = [
        ["g++", "-O3", "-std=c++17", "-fPIC", "-Wall", "-Wextra", "-pthread", "-c",
         os.path.join(CSRC, "encode.cpp"), "-o", enc_o],
        [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "-c", os.path.join(CSRC, "decode.cu"), "-o", dec_o],
        [NVCC, *ARCH, "-shared", "-o", LIB, enc_o, dec_o, "-lpthread"],
    ]
    for c in cmds:
        r = subprocess.run(c, capture_output=True, text=True)
        if verbose or r.returncode:
            sys.stderr.write(" ".join(c) + "\n" + r.stdout + r.stderr)
        if r.returncode:
            raise RuntimeError(f"build failed: {' '.join(c)}")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
