"""Bounds-checking build (stands in for compute-sanitizer memcheck, which this GPU pool has
disabled): libmc.so rebuilt with -DMC_CHECK_BOUNDS=1 range-checks every output store
(index, vertex, quantized buffers), every staged-record read of a valid record (flag
words, index / reuse bytes, attribute bits), the N[] and pivot indices and every TMA
staging size, and traps on a violation.  tests/sanitize_decode.py runs the sanitizer
workloads (cfg1 in three codecs x two index formats, every GTS-Reuse stream with T' <= 5,
long fans with 32-lane groups, bit-reader and generic layouts, culled decode, the static-
stride and dynamic-claim kernels) plus 40 rounds of random record corruption through that
build in a subprocess: it must exit 0 with no check failure."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bounds_checking_build(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    sys.path.insert(0, ROOT)
    from paper_2404_06359_b200 import _build
    lib = str(tmp_path / "libmc_bounds.so")
    _build.build(force=True, lib=lib, extra_flags=["-DMC_CHECK_BOUNDS=1"], bdir=str(tmp_path / "obj"))
    env = dict(os.environ, MC_LIB=lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "sanitize_decode.py"), "--big", "--fuzz"],
                       capture_output=True, text=True, timeout=1200, cwd=ROOT, env=env)
    out = r.stdout + r.stderr
    assert "bounds check failed" not in out, out[-4000:]
    assert r.returncode == 0, out[-4000:]
    assert "decode error bits: 0" in out and "fuzz rounds: 40" in out, out[-4000:]
