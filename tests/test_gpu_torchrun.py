"""GPU: bench.py launched the way the driver launches multi-GPU runs (torch.distributed.run,
one process per rank), here with 2 ranks sharing the one GPU of the box (collectives on
gloo host copies; on an 8-GPU box every rank has its own GPU and NCCL).  Both scaling modes
must produce one JSON line whose all-reduced checksums equal the oracle's decode of the
whole scene (strong: one city split over the ranks; weak: one city block per rank)."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("scaling", ["strong", "weak"])
def test_torchrun_two_ranks(orc, scaling):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    sys.path.insert(0, ROOT)
    import bench
    import paper_2404_06359_b200 as mc
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
           "--steps", "4", "--warmup", "3", "--instances", "6", "--prototypes", "3", "--scaling", scaling,
           "--no-e2e", "--no-cpu-baseline", "--sustained-seconds", "0"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == scaling and d["checksum"]["error_bits"] == 0
    assert d["value"] > 0 and d["config"]["n_ranks"] == 2
    full, _ = bench.build_blob(mc, "cfg4_city", 0, 1, 2, 6 if scaling == "strong" else 12, protos_k=(3, 91))
    err, errs, idx, q, f = orc.decode(np.array(full.bytes), want_q=False)
    assert err == 0
    assert d["checksum"]["indices"] == orc.checksum(idx, 0)
    assert d["checksum"]["vertices"] == orc.checksum(f, 0)
