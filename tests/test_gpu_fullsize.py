"""Full-size parity: BASELINE cfg4 (the instanced city, 1000 instances of 256 seeded
buildings, ~99.2M triangles, ~1.14M records) decoded by exactly the kernel and launch
configuration bench.py times, checked against the oracle:

  - 512 sampled records element by element (indices, fp32 bit patterns) against the
    oracle's sequential decode of those records;
  - the WHOLE outputs through FORMAT.md §6 checksums: the oracle decodes every record on
    host threads and checksums its buffers; the GPU's timed-kernel outputs are copied
    back and checksummed with the same (oracle) routine; the stats kernel's device
    checksums must match too.
"""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


@pytest.fixture(scope="module")
def mc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2404_06359_b200 as mc
    mc.lib()
    return mc


def test_cfg4_city_full_size(mc, orc):
    import bench
    blob, meta = bench.build_blob(mc, "cfg4_city", 0, 1, 2, 1000)
    data = np.array(blob.bytes)
    L = blob.layout
    assert L.num_meshlets > 1_100_000 and 95_000_000 < L.total_t < 105_000_000
    db = mc.DeviceBlob(blob, want_vertices=True, want_quantized=False)
    stream = torch.cuda.current_stream()
    db.decode(stream=stream)                                   # the timed kernel
    torch.cuda.synchronize()
    gi = db.indices.cpu().numpy().view(np.uint32)
    gf = db.vertices.cpu().numpy().view(np.uint32)
    st = db.decode_stats(stream=stream)                        # the stats kernel
    assert st["error_bits"] == 0 and st["triangles"] == L.total_tp and st["vertices"] == L.total_v

    # sampled records, element by element
    rng = np.random.default_rng(0)
    for m in np.sort(rng.choice(L.num_meshlets, 512, replace=False)):
        err, meta_m, tri, q, f = orc.decode_meshlet(data, int(m), want_q=False)
        assert err == 0
        vb, tb, V, Tp = (int(x) for x in meta_m[:4])
        np.testing.assert_array_equal(gi[3 * tb:3 * (tb + Tp)], (tri.reshape(-1) + vb).astype(np.uint32))
        np.testing.assert_array_equal(gf[L.n_out * vb:L.n_out * (vb + V)], f.reshape(-1).view(np.uint32))

    # the whole outputs, through checksums of the oracle's own full decode
    info = orc.blob_info(data)
    idx = np.zeros(3 * info.total_tp, np.uint32)
    fo = np.zeros(info.n_out * info.total_v, np.float32)
    cores = max(1, min(32, len(os.sched_getaffinity(0))))
    bounds = np.linspace(0, info.M, 8 * cores + 1).astype(np.int64)
    with ThreadPoolExecutor(cores) as ex:
        errs = list(ex.map(lambda i: orc.decode_range_raw(data, int(bounds[i]), int(bounds[i + 1]), idx, None, fo),
                           range(len(bounds) - 1)))
    assert all(e == 0 for e in errs)
    cs_i, cs_f = orc.checksum(idx, 0), orc.checksum(fo, 0)
    assert orc.checksum(gi, 0) == cs_i and orc.checksum(gf, 0) == cs_f
    assert st["checksum_indices"] == cs_i and st["checksum_vertices"] == cs_f
