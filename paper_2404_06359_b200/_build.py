"""Build libmc.so in-tree: host encoder (g++) + sm_100a decode kernels (nvcc).

    python -m paper_2404_06359_b200._build [--force] [-v]

The decode kernel family is instantiated in six units (decode_inst.cu compiled with
-DMC_INST_CODEC={1,2,3} x -DMC_INST_STATS={0,1}) plus the host unit decode.cu; all units
and the encoder compile in parallel.  Extra nvcc flags (experiments): MC_NVCC_FLAGS.
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
SOURCES = [os.path.join(CSRC, f) for f in ("encode.cpp", "decode.cu", "decode_inst.cu", "decode_kernel.cuh", "oct_math.cuh")] + \
          [os.path.join(ROOT, "include", "mc.h")]
INSTS = [(c, st) for c in (1, 2, 3) for st in (0, 1)]


def _stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    return any(os.path.getmtime(s) > t for s in SOURCES)


def _nvcc(src, out, extra):
    return [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v", *extra,
            "-c", src, "-o", out]


def build(force: bool = False, verbose: bool = False, lib: str = LIB, extra_flags=None, bdir=None) -> str:
    if not force and not _stale(lib):
        return lib
    extra = list(extra_flags) if extra_flags is not None else os.environ.get("MC_NVCC_FLAGS", "").split()
    bdir = bdir or os.path.join(PKG, "build")
    os.makedirs(bdir, exist_ok=True)
    enc_o = os.path.join(bdir, "encode.o")
    host_o = os.path.join(bdir, "decode.o")
    inst_o = [os.path.join(bdir, f"decode_inst_{c}_{st}.o") for c, st in INSTS]
    jobs = [["g++", "-O3", "-std=c++17", "-fPIC", "-Wall", "-Wextra", "-pthread", "-c",
             os.path.join(CSRC, "encode.cpp"), "-o", enc_o],
            _nvcc(os.path.join(CSRC, "decode.cu"), host_o, extra)]
    jobs += [_nvcc(os.path.join(CSRC, "decode_inst.cu"), o, extra + [f"-DMC_INST_CODEC={c}", f"-DMC_INST_STATS={st}"])
             for (c, st), o in zip(INSTS, inst_o)]
    procs = [(c, subprocess.Popen(c, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)) for c in jobs]
    failed = None
    for c, p in procs:
        out, err = p.communicate()
        if verbose or p.returncode:
            sys.stderr.write(" ".join(c) + "\n" + out + err)
        if p.returncode and failed is None:
            failed = c
    if failed:
        raise RuntimeError(f"build failed: {' '.join(failed)}")
    link = [NVCC, *ARCH, "-shared", "-o", lib, enc_o, host_o, *inst_o, "-lpthread"]
    r = subprocess.run(link, capture_output=True, text=True)
    if verbose or r.returncode:
        sys.stderr.write(" ".join(link) + "\n" + r.stdout + r.stderr)
    if r.returncode:
        raise RuntimeError(f"build failed: {' '.join(link)}")
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
