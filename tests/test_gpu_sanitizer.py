"""compute-sanitizer gate: memcheck, racecheck and synccheck over the decode
of cfg1, the exhaustive tiny GTS-Reuse streams, long multi-word fans, a generic layout,
a culled decode, the static-stride kernel and (memcheck only) a dynamic-claim launch —
0 errors.  Runs tests/sanitize_decode.py under each tool."""
import os
import re
import shutil
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_sanitizer_clean(tool):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.exists(SAN):
        pytest.skip("compute-sanitizer not found")
    cmd = [SAN, "--tool", tool, "--error-exitcode", "99", "--print-limit", "20"]
    if tool == "memcheck":
        cmd += ["--leak-check", "no"]
    args = [sys.executable, os.path.join(ROOT, "tests", "sanitize_decode.py")] + (["--big"] if tool == "memcheck" else [])
    r = subprocess.run(cmd + args, capture_output=True, text=True, timeout=1500, cwd=ROOT)
    out = r.stdout + r.stderr
    if tool == "racecheck":   # "RACECHECK SUMMARY: N hazards displayed (E errors, W warnings)"
        m = re.search(r"RACECHECK SUMMARY: (\d+) hazards? displayed \((\d+) errors?, (\d+) warnings?\)", out)
        assert m is not None or "ERROR SUMMARY: 0 errors" in out, out[-3000:]
        if m is not None:
            assert int(m.group(2)) == 0 and int(m.group(3)) == 0, out[:6000]
    else:
        m = re.search(r"ERROR SUMMARY: (\d+) error", out)
        assert m is not None, out[-3000:]
        assert int(m.group(1)) == 0, out[:6000]
    assert r.returncode == 0, out[-3000:]
