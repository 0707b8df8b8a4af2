"""GPU parity for the Basic codec (codec 3) and the local u8x4 index output.

Same bar as tests/test_gpu_parity.py: indices bit-exact, fp32 attributes 0 ULP, checksums
equal the oracle's (FORMAT.md §6), for both the stats and the timed kernels.  Expected
values come only from oracle/ (sequential decode, oracle encoder) — never from the CUDA path.
"""
import numpy as np
import pytest

import synth
from streams import basic_meshlet, pack_meshlets

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


def check(mc, orc, blob, index_format="u32", want_q=True):
    blob = np.ascontiguousarray(blob)
    L = mc.parse_header(blob)
    db = mc.DeviceBlob(blob, want_vertices=True, want_quantized=want_q, index_format=index_format)
    st = db.decode_stats()
    torch.cuda.synchronize()
    err, errs, idx, q, f = orc.decode(blob, want_q=want_q)
    assert err == 0 and st["error_bits"] == 0, (err, st)
    if index_format == "u8x4":
        e8, want = orc.decode_u8x4(blob)
        assert e8 == 0
        np.testing.assert_array_equal(_u32(db.indices), want)
        assert st["checksum_indices"] == orc.checksum(want, L.base_tri)
    else:
        np.testing.assert_array_equal(_u32(db.indices), idx)
        assert st["checksum_indices"] == orc.checksum(idx, 3 * L.base_tri)
    np.testing.assert_array_equal(_u32(db.vertices), f.view(np.uint32))
    assert st["checksum_vertices"] == orc.checksum(f, L.n_out * L.base_vtx)
    if want_q:
        np.testing.assert_array_equal(_u32(db.quantized), q)
    tri = idx.reshape(-1, 3)
    deg = (tri[:, 0] == tri[:, 1]) | (tri[:, 1] == tri[:, 2]) | (tri[:, 0] == tri[:, 2])
    assert st["degenerate"] == int(deg.sum()) and st["triangles"] == L.total_tp
    # the timed kernel writes the same bytes
    db2 = mc.DeviceBlob(blob, want_vertices=True, want_quantized=want_q, index_format=index_format)
    db2.decode()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(_u32(db2.indices), _u32(db.indices))
    np.testing.assert_array_equal(_u32(db2.vertices), _u32(db.vertices))
    return db, st


@pytest.mark.parametrize("limits", [(64, 126), (128, 256), (32, 32), (256, 256), (3, 1)])
def test_basic_oracle_encoded_grid(mc, orc, limits):
    check(mc, orc, orc.encode(synth.quad_grid(), *limits, 3).blob)


@pytest.mark.parametrize("seed", range(4))
def test_basic_random_patches_generic_layout(mc, orc, seed):
    check(mc, orc, orc.encode(synth.random_patch(seed), 64, 126, 3).blob)


def test_basic_product_encoded(mc, orc):
    for m, lim in [(synth.torus(300, 150), (64, 126)), (synth.displaced_sphere(60), (128, 256)),
                   (synth.displaced_sphere(40, oct_normals=False).with_bits(10), (64, 126))]:
        b = mc.mc_encode(m, *lim, mc.MC_CODEC_BASIC)
        check(mc, orc, np.array(b.bytes))


@pytest.mark.parametrize("codec", [1, 2, 3])
@pytest.mark.parametrize("limits", [(64, 126), (128, 256), (256, 256)])
def test_u8x4_all_codecs(mc, orc, codec, limits):
    for m in (synth.quad_grid(), synth.displaced_sphere(30), synth.random_patch(9, 30, 20)):
        b = mc.mc_encode(m, *limits, codec)
        check(mc, orc, np.array(b.bytes), index_format="u8x4", want_q=False)


def test_u8x4_city_shard(mc, orc):
    """An instance-range shard (non-zero base_tri / base_vtx): u8x4 words and their
    checksum keep global word positions (FORMAT.md §6)."""
    scene = synth.city(num_instances=6, num_prototypes=2, k=12)
    protos = [mc.mc_encode(p, 64, 126, 2) for p in scene.prototypes]
    blob = mc.mc_blob_instance_range(protos, scene.instance_proto, scene.instance_offset, 2, 3)
    check(mc, orc, np.array(blob.bytes), index_format="u8x4", want_q=False)


def test_basic_malformed(mc, orc):
    """FORMAT.md §5 for Basic: index >= V -> INDEX, R != 0 -> COUNTS; the stats kernel
    reports what the oracle reports."""
    good = basic_meshlet(4, [(0, 1, 2), (2, 1, 3)])
    bad_idx = basic_meshlet(3, [(0, 1, 2), (2, 1, 3)])
    for ms, R, want in (([good, bad_idx], [0, 0], orc.DERR_INDEX), ([good, good], [0, 1], orc.DERR_COUNTS)):
        blob = pack_meshlets(orc, 3, ms, R=R)
        err, errs, idx, q, f = orc.decode(blob)
        db = mc.DeviceBlob(blob)
        st = db.decode_stats()
        assert err == want and st["error_bits"] == want and st["first_bad_meshlet"] == 1


def test_u8x4_buffer_size_checked(mc, orc):
    b = orc.encode(synth.quad_grid(4, 4), 64, 126, 2).blob
    L = mc.parse_header(b)
    d_blob = torch.from_numpy(np.array(b)).cuda()
    small = torch.empty(L.total_tp - 1, dtype=torch.int32, device="cuda")
    with pytest.raises(mc.MCError):
        mc.mc_decode_meshlets(L, d_blob, small, flags=mc.MC_DECODE_INDEX_LOCAL_U8X4)
    ok = torch.empty(L.total_tp, dtype=torch.int32, device="cuda")
    mc.mc_decode_meshlets(L, d_blob, ok, flags=mc.MC_DECODE_INDEX_LOCAL_U8X4)
    with pytest.raises(mc.MCError):
        mc.mc_decode_meshlets(L, d_blob, ok, flags=0)   # u32 output needs 3 words per triangle
