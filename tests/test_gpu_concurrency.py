"""GPU: decodes of different kernel variants in flight at the same time on two streams,
with the library work pool (d_work = NULL) and with caller work buffers, stay bit-exact
with the oracle; the work buffer is left zeroed by every decode (include/mc.h d_work)."""
import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2404_06359_b200 as mc
    mc.lib()
    return mc


def _u32(t):
    return t.cpu().numpy().view(np.uint32)


@pytest.fixture(scope="module")
def blobs(mc):
    # four kernel variants: GTS n=7 oct, GTS-Reuse n=3, Basic n=8, GTS-Reuse generic widths
    m1 = synth.displaced_sphere(60)
    m2 = synth.torus(300, 150)
    m3 = synth.displaced_sphere(50, oct_normals=False)
    m4 = synth.random_patch(3, nx=120, ny=90)
    return [mc.mc_encode(m1, 64, 126, 1), mc.mc_encode(m2, 64, 126, 2), mc.mc_encode(m3, 64, 126, 3),
            mc.mc_encode(m4, 128, 256, 2)]


@pytest.mark.parametrize("work", ["pool", "caller"])
def test_concurrent_variants_two_streams(mc, orc, blobs, work):
    dbs = [mc.DeviceBlob(b, want_vertices=True, want_quantized=True) for b in blobs]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    torch.cuda.synchronize()
    for rep in range(6):
        for i, db in enumerate(dbs):
            # pool: a blob's decodes alternate streams (launches of every variant overlap,
            # each on its own pool block; repeated decodes of one blob write equal bytes);
            # caller: a blob keeps one stream, so its work buffer is reused in order
            s = streams[(i + rep) % 2] if work == "pool" else streams[i % 2]
            mc.mc_decode_meshlets(db.layout, db.d_blob, db.indices, db.vertices, db.quantized, stream=s,
                                  d_work=db.work if work == "caller" else None)
    torch.cuda.synchronize()
    for b, db in zip(blobs, dbs):
        err, errs, idx, q, f = orc.decode(np.array(b.bytes))
        assert err == 0
        np.testing.assert_array_equal(_u32(db.indices), idx)
        np.testing.assert_array_equal(_u32(db.quantized), q)
        np.testing.assert_array_equal(_u32(db.vertices), f.view(np.uint32))
        assert not _u32(db.work).any(), "work buffer must be left zeroed"


def test_pool_more_launches_than_blocks(mc, orc, blobs):
    """Far more pool-backed launches than pool blocks, ordered on one stream: every block is
    reused many times and must be zero each time (self-reset, no memset)."""
    b = blobs[1]
    db = mc.DeviceBlob(b, want_vertices=True)
    for _ in range(200):
        mc.mc_decode_meshlets(db.layout, db.d_blob, db.indices, db.vertices)
    torch.cuda.synchronize()
    err, errs, idx, q, f = orc.decode(np.array(b.bytes), want_q=False)
    np.testing.assert_array_equal(_u32(db.indices), idx)
    np.testing.assert_array_equal(_u32(db.vertices), f.view(np.uint32))


def test_misaligned_or_small_work_rejected(mc, blobs):
    db = mc.DeviceBlob(blobs[0])
    with pytest.raises(mc.MCError):
        mc.mc_decode_meshlets(db.layout, db.d_blob, db.indices, db.vertices, d_work=db.work[:10])
    w = torch.zeros(mc.MC_DECODE_WORK_WORDS * 4 + 4, dtype=torch.uint8, device="cuda")[1:]
    with pytest.raises(mc.MCError):
        mc.mc_decode_meshlets(db.layout, db.d_blob, db.indices, db.vertices, d_work=w)
