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
    # racecheck counts its (TMA false-positive) warnings in the exit code: its hazards are
    # parsed below instead
    cmd = [SAN, "--tool", tool, "--print-limit", "20"] + ([] if tool == "racecheck" else ["--error-exitcode", "99"])
    if tool in ("racecheck", "synccheck"):   # 8-lane groups: 32 groups x 2 mbarriers per CTA
        cmd += ["--num-cuda-barriers", "128"]
    if tool == "memcheck":
        cmd += ["--leak-check", "no"]
    args = [sys.executable, os.path.join(ROOT, "tests", "sanitize_decode.py")] + (["--big"] if tool == "memcheck" else [])
    r = subprocess.run(cmd + args, capture_output=True, text=True, timeout=1500, cwd=ROOT)
    out = r.stdout + r.stderr
    if "compute-sanitizer is closed" in out:
        # the GPU pool's operators disabled the tool (a wrapper prints this and runs nothing);
        # the committed logs under profiles/round2/ hold the last sanitizer runs
        pytest.skip("compute-sanitizer disabled on this GPU pool")
    if tool == "racecheck":   # "RACECHECK SUMMARY: N hazards displayed (E errors, W warnings)"
        m = re.search(r"RACECHECK SUMMARY: (\d+) hazards? displayed \((\d+) errors?, (\d+) warnings?\)", out)
        assert m is not None or "ERROR SUMMARY: 0 errors" in out, out[-3000:]
        if m is not None:
            assert int(m.group(2)) == 0, out[:6000]
            # racecheck does not model TMA completion (cp.async.bulk ... mbarrier::complete_tx
            # + mbarrier.try_wait): it reports the bulk copy's shared-memory writes against the
            # reads that follow the wait as WARNINGS.  Every warning must be exactly that pair;
            # any other hazard fails.  (With the records staged through the generic proxy
            # instead, -DMC_GENERIC_COPY=1, racecheck reports 0 hazards: profiles/round2/.)
            blocks = re.findall(r"(Warning|Error): Race reported between (\w+) access at (\S+)", out)
            assert blocks, out[:6000]
            for kind, acc, where in blocks:
                assert kind == "Warning" and acc == "Write" and "bulk_g2s" in where, (kind, acc, where)
    else:
        m = re.search(r"ERROR SUMMARY: (\d+) error", out)
        assert m is not None, out[-3000:]
        assert int(m.group(1)) == 0, out[:6000]
    assert r.returncode == 0, out[-3000:]
