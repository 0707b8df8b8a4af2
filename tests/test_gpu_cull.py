"""GPU parity for the cone-culled, compacted decode (FORMAT.md §1.5, §7).

The sm_100a path (cull reduce / tile scan / emit kernels, then the decode kernel over the
visible-record list) against the oracle's sequential culled decode: the same visible
set and counts, compacted indices bit-exact (u32 and u8x4), q bit-exact, floats 0 ULP,
checksums equal, for product-made cones and for hand-set cull tables (oracle-inserted).
"""
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


def _dirs(seed, k=5):
    rng = np.random.default_rng(seed)
    d = rng.normal(size=(k, 3))
    return (d / np.linalg.norm(d, axis=1, keepdims=True)).astype(np.float32)


def check_culled(mc, orc, blob, d, index_format="u32", want_q=True):
    blob = np.ascontiguousarray(blob)
    u8 = index_format == "u8x4"
    err, vis, c, idx, q, f = orc.decode_culled(blob, d, u8x4=u8, want_q=want_q)
    assert err == 0
    db = mc.DeviceBlob(blob, want_vertices=True, want_quantized=want_q, index_format=index_format)
    st = db.decode_culled(d, stats=True)
    got = db.read_cull_counts()
    assert got == c, (got, c)
    L = db.layout
    nidx = (1 if u8 else 3) * c["Tp"]
    np.testing.assert_array_equal(_u32(db.indices)[:nidx], idx)
    np.testing.assert_array_equal(_u32(db.vertices)[:L.n_out * c["V"]], f.view(np.uint32))
    if want_q:
        np.testing.assert_array_equal(_u32(db.quantized)[:L.n * c["V"]], q)
    assert st["error_bits"] == 0 and st["triangles"] == c["Tp"] and st["vertices"] == c["V"]
    assert st["checksum_indices"] == orc.checksum(idx, 0)
    assert st["checksum_vertices"] == orc.checksum(f, 0)
    # the timed kernels (no stats) write the same bytes
    db2 = mc.DeviceBlob(blob, want_vertices=True, want_quantized=want_q, index_format=index_format)
    db2.decode_culled(d)
    torch.cuda.synchronize()
    assert db2.read_cull_counts() == c
    np.testing.assert_array_equal(_u32(db2.indices)[:nidx], idx)
    np.testing.assert_array_equal(_u32(db2.vertices)[:L.n_out * c["V"]], f.view(np.uint32))
    return c


@pytest.mark.parametrize("codec", [1, 2, 3])
def test_culled_product_cones(mc, orc, codec):
    for mesh, lim in [(synth.displaced_sphere(40), (64, 126)), (synth.quad_grid(), (32, 32)),
                      (synth.displaced_sphere(30, oct_normals=False).with_bits(11), (128, 256))]:
        b = np.array(mc.mc_encode(mesh, *lim, codec, cull_cones=True).bytes)
        seen = 0
        for d in _dirs(codec):
            c = check_culled(mc, orc, b, d)
            seen += c["records"]
        assert 0 < seen < 5 * mc.parse_header(b).num_meshlets          # some culled, some kept


def test_culled_u8x4_and_vw(mc, orc):
    m = synth.displaced_sphere(36)
    b = np.array(mc.mc_encode(m, 64, 126, 2, cull_cones=True, variable_widths=True).bytes)
    for d in _dirs(11, 3):
        check_culled(mc, orc, b, d, index_format="u8x4", want_q=False)
        check_culled(mc, orc, b, d)


def test_culled_handset_tables(mc, orc):
    """Oracle-inserted tables: never, always, random subsets, the exact decision boundary;
    more than one cull tile (2048 records) so the tile scan carries across tiles."""
    m = synth.torus(300, 150)
    blob = np.array(mc.mc_encode(m, 32, 32, 2).bytes)
    M = mc.parse_header(blob).num_meshlets
    assert M > 2048                     # at least two cull tiles
    rng = np.random.default_rng(5)
    d = np.array([0.0, 0.6, 0.8], np.float32)
    tables = {"never": np.tile([0, 0, 1, 2.0], (M, 1)), "always": np.tile([0, 0.6, 0.8, -2.0], (M, 1))}
    sub = np.zeros((M, 4), np.float32)
    sub[:, :3] = d
    sub[:, 3] = np.where(rng.random(M) < 0.5, 0.5, 2.0)
    tables["subset"] = sub
    edge = np.zeros((M, 4), np.float32)
    edge[:, 0] = 1.0
    edge[:, 3] = np.where(np.arange(M) % 3 == 0, np.float32(1.0), np.nextafter(np.float32(1.0), np.float32(0)))
    tables["boundary"] = edge
    for name, t in tables.items():
        cb = orc.add_cull(blob, t)
        dd = np.array([1, 0, 0], np.float32) if name == "boundary" else d
        c = check_culled(mc, orc, cb, dd)
        if name == "never":
            assert c["records"] == M
        if name == "always":
            assert c["records"] == 0


def test_culled_city_instances(mc, orc):
    scene = synth.city(num_instances=8, num_prototypes=3, k=16)
    protos = [mc.mc_encode(p, 64, 126, 2, cull_cones=True) for p in scene.prototypes]
    inst = np.array(mc.mc_blob_instance_range(protos, scene.instance_proto, scene.instance_offset, 2, 5).bytes)
    for d in _dirs(3, 3):
        check_culled(mc, orc, inst, d)


def test_culled_requires_table(mc, orc):
    b = orc.encode(synth.quad_grid(8, 8), 64, 126, 2).blob
    db = mc.DeviceBlob(b)
    with pytest.raises(mc.MCError):
        db.decode_culled([0, 0, 1])
