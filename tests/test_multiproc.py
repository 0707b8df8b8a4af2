"""Multi-process (gloo, world size 2, CPU) check of the sharded path bench.py runs under
torchrun: each rank builds its instance-range shard of the city (strong: a split of one
city; weak: its own block of an N-times larger city), decodes it (here with the oracle, on
CPU; tests/test_gpu_multiproc.py runs the product), and the checksum all-reduce reproduces
the whole scene's checksum."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

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
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    import oracle
    import paper_2404_06359_b200 as mc
    blob, meta = bench.build_blob(mc, "cfg4_city", rank, world, 2, instances=3, protos_k=(2, 6), scaling=scaling)
    data = np.array(blob.bytes)
    err, errs, idx, qv, f = oracle.decode(data)
    L = blob.layout
    local = [oracle.checksum(idx, 3 * L.base_tri), oracle.checksum(f, L.n_out * L.base_vtx)]
    total = bench.allreduce_u64_sum(local, dist, "cpu")
    tri = torch.tensor([float(L.total_t)])
    dist.all_reduce(tri)
    q.put((rank, err, local, total, float(tri.item()), L.base_tri, L.total_tp))
    dist.destroy_process_group()


@pytest.mark.parametrize("scaling", ["strong", "weak"])
def test_two_rank_shards_checksum_allreduce(orc, scaling):
    import bench
    import paper_2404_06359_b200 as mc
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, scaling, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # the whole scene, built once on one process
    full, _ = bench.build_blob(mc, "cfg4_city", 0, 1, 2, instances=3 if scaling == "strong" else 6, protos_k=(2, 6))
    err, errs, idx, qv, f = orc.decode(np.array(full.bytes))
    L = full.layout
    want = [orc.checksum(idx, 0), orc.checksum(f, 0)]
    assert all(r[1] == 0 for r in res)
    assert res[0][3] == res[1][3] == want
    assert res[0][4] == float(L.total_t)
    # rank shards tile the scene: rank 1 starts where rank 0 ends
    assert res[1][5] == res[0][5] + res[0][6]
