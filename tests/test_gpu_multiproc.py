"""GPU: the sharded product path under two processes (gloo, world size 2) that share
cuda:0.  Each rank builds its instance-range shard of the city (bench.build_blob, strong
and weak splits), decodes it with the PRODUCT (sm_100a kernel through the C ABI), and the
all-reduced checksums equal the whole scene's oracle checksums (FORMAT.md §6)."""
import os
import socket

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


def _worker(rank, world, port, scaling, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    import paper_2404_06359_b200 as mc
    torch.cuda.set_device(0)
    blob, meta = bench.build_blob(mc, "cfg4_city", rank, world, 2, instances=4, protos_k=(3, 8), scaling=scaling)
    db = mc.DeviceBlob(blob, device="cuda:0", want_vertices=True)
    db.decode()
    st = db.decode_stats()
    local = [st["checksum_indices"], st["checksum_vertices"]]
    total = bench.allreduce_u64_sum(local, dist, "cpu")
    q.put((rank, st["error_bits"], total, blob.layout.total_t, blob.layout.base_tri, blob.layout.total_tp))
    dist.destroy_process_group()


@pytest.mark.parametrize("scaling", ["strong", "weak"])
def test_two_ranks_share_gpu_product_decode(orc, scaling):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import bench
    import paper_2404_06359_b200 as mc
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, scaling, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    # the whole scene on one process, decoded by the oracle
    n_inst = 4 if scaling == "strong" else 8
    full, _ = bench.build_blob(mc, "cfg4_city", 0, 1, 2, instances=n_inst, protos_k=(3, 8))
    err, errs, idx, qv, f = orc.decode(np.array(full.bytes), want_q=False)
    want = [orc.checksum(idx, 0), orc.checksum(f, 0)]
    assert err == 0 and all(r[1] == 0 for r in res)
    assert res[0][2] == res[1][2] == want
    assert res[0][3] + res[1][3] == full.layout.total_t
    assert res[1][4] == res[0][4] + res[0][5]      # rank 1's triangles follow rank 0's
