"""CPU checks of the C ABI boundary: libmc.so loads, exports every function include/mc.h
declares, and its host-side calls (encoder, header parse, shards, extract, instancing)
behave; no GPU compute is called here."""
import os
import re

import numpy as np
import pytest

import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def mc():
    from paper_2404_06359_b200 import _build
    _build.build()
    import paper_2404_06359_b200 as mc
    mc.lib()
    return mc


def test_exports_every_declared_symbol(mc):
    hdr = open(os.path.join(ROOT, "include", "mc.h")).read()
    code = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    declared = set(re.findall(r"\b(mc_[a-z_0-9]+)\s*\(", code))
    assert "mc_decode_meshlets" in declared and "mc_encode" in declared
    L = mc.lib()
    for name in sorted(declared):
        assert hasattr(L, name), name
    assert L.mc_abi_version() == 4
    out = os.popen(f"nm -D {mc.LIB_PATH}").read()
    for name in declared:
        assert re.search(rf"\bT {name}\b", out), name


def test_sm100a_code_present(mc):
    sass = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {mc.LIB_PATH} 2>&1").read()
    assert "sm_100a" in sass


def test_status_and_errors(mc):
    with pytest.raises(mc.MCError):
        mc.parse_header(np.zeros(200, np.uint8))
    m = synth.quad_grid(2, 2)
    bad = synth.Mesh(m.indices.copy(), m.attributes, m.bits, m.semantic)
    bad.indices[0, 0] = bad.indices[0, 1]
    with pytest.raises(mc.MCError, match="invalid source mesh"):
        mc.mc_encode(bad)
    with pytest.raises(mc.MCError, match="limits"):
        mc.mc_encode(m, 300, 126)
    bad2 = synth.Mesh(m.indices.copy(), m.attributes, m.bits, m.semantic)
    bad2.indices[0, 0] = 10**6
    with pytest.raises(mc.MCError):
        mc.mc_encode(bad2)


def test_product_encoder_roundtrip_via_oracle(mc, orc):
    """Oracle decode of mc_encode output recovers the source triangles (winding kept) and
    the attributes within Δ/2 — the oracle checking the product encoder."""
    for mesh, lim in [(synth.quad_grid(), (64, 126)), (synth.displaced_sphere(16), (128, 256)),
                      (synth.random_patch(7), (32, 32)), (synth.torus(50, 30), (256, 256)),
                      (synth.random_patch(8), (16, 8))]:
        for codec in (1, 2, 3):
            b = mc.mc_encode(mesh, *lim, codec)
            err, errs, idx, q, f = orc.decode(np.array(b.bytes))
            assert err == 0
            sv, st = b.source_map()
            tri = idx.reshape(-1, 3).astype(np.int64)
            g = sv[tri]
            deg = (tri[:, 0] == tri[:, 1]) | (tri[:, 1] == tri[:, 2]) | (tri[:, 0] == tri[:, 2])
            assert np.array_equal(synth.canonical_triangles(g[~deg]), synth.canonical_triangles(mesh.indices))
            assert deg.sum() == 4 * b.encode_stats()["restarts"]
            assert np.all((st == 0xFFFFFFFF) == deg)
            if codec == 3:   # Basic: no restarts, T' = T
                assert b.encode_stats()["restarts"] == 0 and b.layout.total_tp == len(mesh.indices)
            L = b.layout
            assert L.v_max == lim[0] and L.t_max == lim[1]
            from streams import read_records
            for r in read_records(np.array(b.bytes)):
                assert 3 <= r["V"] <= lim[0] and r["Tp"] <= lim[1]


def test_shards_and_extract(mc, orc):
    b = mc.mc_encode(synth.torus(80, 40), 64, 126, 2)
    ranges = b.shard_ranges(5)
    assert sum(c for _, c in ranges) == b.layout.num_meshlets
    assert [f for f, _ in ranges] == sorted(f for f, _ in ranges)
    full = orc.decode(np.array(b.bytes))
    for f0, c in ranges:
        s = b.extract(f0, c)
        err, errs, idx, q, fl = orc.decode(np.array(s.bytes))
        assert err == 0
        L = s.layout
        assert np.array_equal(idx, full[2][3 * L.base_tri:3 * (L.base_tri + L.total_tp)])
        assert np.array_equal(q, full[3][L.n * L.base_vtx:L.n * (L.base_vtx + L.total_v)])


def test_instance(mc, orc):
    scene = synth.city(num_instances=6, num_prototypes=2, k=6)
    protos = [mc.mc_encode(p, 64, 126, 2) for p in scene.prototypes]
    city = mc.mc_blob_instance(protos, scene.instance_proto, scene.instance_offset)
    L = city.layout
    assert L.num_objects == 6
    assert L.total_t == scene.num_triangles
    err, errs, idx, q, f = orc.decode(np.array(city.bytes))
    assert err == 0
    # instance i decodes to its prototype shifted by the instance offset (positions)
    off_v = 0
    for i, p in enumerate(scene.instance_proto):
        pl = protos[p].layout
        pe = orc.decode(np.array(protos[p].bytes))
        fi = f.reshape(-1, L.n_out)[off_v:off_v + pl.total_v]
        fp = pe[4].reshape(-1, L.n_out)
        assert np.allclose(fi[:, :3], fp[:, :3] + scene.instance_offset[i], atol=1e-3)
        assert np.array_equal(fi[:, 3:], fp[:, 3:])
        off_v += pl.total_v


def test_instance_range_shards(mc, orc):
    """Instance-range shards carry global bases: their outputs and checksums tile the
    whole scene's (the weak-scaling multi-GPU layout)."""
    scene = synth.city(num_instances=7, num_prototypes=3, k=5, seed=2)
    protos = [mc.mc_encode(p, 64, 126, 2) for p in scene.prototypes]
    full = mc.mc_blob_instance(protos, scene.instance_proto, scene.instance_offset)
    fe = orc.decode(np.array(full.bytes))
    cs = 0
    for first, cnt in ((0, 3), (3, 1), (4, 3)):
        s = mc.mc_blob_instance_range(protos, scene.instance_proto, scene.instance_offset, first, cnt)
        L = s.layout
        err, errs, idx, q, f = orc.decode(np.array(s.bytes))
        assert err == 0
        np.testing.assert_array_equal(idx, fe[2][3 * L.base_tri:3 * (L.base_tri + L.total_tp)])
        np.testing.assert_array_equal(f.view(np.uint32),
                                      fe[4].view(np.uint32)[L.n_out * L.base_vtx:L.n_out * (L.base_vtx + L.total_v)])
        cs = (cs + orc.checksum(idx, 3 * L.base_tri)) % 2**64
    assert cs == orc.checksum(fe[2], 0)


@pytest.mark.parametrize("codec", [1, 2, 3])
def test_product_encoder_variable_widths(mc, orc, codec):
    """mc_encode(variable_widths=True) (FORMAT.md VW): the oracle decodes it to exactly the
    values of the fixed-width product blob, and each record's w_c is the bit length of
    its largest code (brute force over the decoded meshlet)."""
    from streams import read_records
    for mesh in (synth.displaced_sphere(20), synth.random_patch(6), synth.torus(40, 20).with_bits(13)):
        fixed = np.array(mc.mc_encode(mesh, 64, 126, codec).bytes)
        var = np.array(mc.mc_encode(mesh, 64, 126, codec, variable_widths=True).bytes)
        assert mc.parse_header(var).flags == 1 and mc.parse_header(fixed).flags == 0
        a, b = orc.decode(fixed), orc.decode(var)
        assert a[0] == 0 and b[0] == 0
        assert np.array_equal(a[2], b[2]) and np.array_equal(a[3], b[3])
        assert np.array_equal(a[4].view(np.uint32), b[4].view(np.uint32))
        n = orc.blob_info(var).n
        q = b[3].reshape(-1, n).astype(np.int64)
        for r in read_records(var):
            codes = q[r["vtx_base"]:r["vtx_base"] + r["V"]] - np.array(r["L"], np.int64)
            for c in range(n):
                assert int(codes[:, c].max()).bit_length() == r["widths"][c] <= mesh.bits[c]


def _backfacing_ok(orc, data, view_dirs):
    """Brute force (FORMAT.md §7 soundness): every real triangle of every culled record
    faces away from the view direction, in double precision from the decoded positions."""
    from streams import read_records
    err, errs, idx, q, f = orc.decode(data, want_q=False)
    assert err == 0
    info = orc.blob_info(data)
    pos = f.reshape(-1, info.n_out)[:, :3].astype(np.float64)
    recs = read_records(data)
    culled = 0
    for d in view_dirs:
        e2, vis, c, *_ = orc.decode_culled(data, d, want_q=False, want_f=False)
        assert e2 == 0
        for r, v in zip(recs, vis):
            if v:
                continue
            tb = r["tri_base"] - info.base_tri
            t = idx[3 * tb:3 * (tb + r["Tp"])].reshape(-1, 3).astype(np.int64) - info.base_vtx
            t = t[(t[:, 0] != t[:, 1]) & (t[:, 1] != t[:, 2]) & (t[:, 0] != t[:, 2])]
            n = np.cross(pos[t[:, 1]] - pos[t[:, 0]], pos[t[:, 2]] - pos[t[:, 0]])
            dots = n @ np.asarray(d, np.float64)
            assert np.all(dots[np.linalg.norm(n, axis=1) > 0] > 0)
            culled += 1
    return culled / (len(view_dirs) * len(recs))


def _dirs(seed, k=12):
    rng = np.random.default_rng(seed)
    d = rng.normal(size=(k, 3))
    return (d / np.linalg.norm(d, axis=1, keepdims=True)).astype(np.float32)


@pytest.mark.parametrize("codec", [1, 2, 3])
def test_product_cull_cones_sound(mc, orc, codec):
    """mc_encode(cull_cones=True): the cones are sound (a culled meshlet is entirely
    back-facing) and useful (a fair share of meshlets culls)."""
    for mesh, lim in [(synth.displaced_sphere(24), (64, 126)), (synth.quad_grid(), (32, 32)),
                      (synth.building(20, 4), (128, 256))]:
        b = mc.mc_encode(mesh, *lim, codec, cull_cones=True)
        data = np.array(b.bytes)
        assert b.layout.flags & 2 and b.layout.off_cull > 0
        frac = _backfacing_ok(orc, data, _dirs(codec))
        assert frac > 0.04


def test_cull_tables_survive_extract_and_instances(mc, orc):
    scene = synth.city(num_instances=4, num_prototypes=2, k=10)
    protos = [mc.mc_encode(p, 64, 126, 2, cull_cones=True) for p in scene.prototypes]
    inst = mc.mc_blob_instance_range(protos, scene.instance_proto, scene.instance_offset, 1, 3)
    data = np.array(inst.bytes)
    assert inst.layout.flags & 2
    _backfacing_ok(orc, data, _dirs(7, 6))                       # translated grids stay sound
    b = mc.mc_encode(synth.displaced_sphere(20), 64, 126, 2, cull_cones=True)
    full = np.array(b.bytes)
    for f0, c in b.shard_ranges(3):
        s = np.array(b.extract(f0, c).bytes)
        d = _dirs(1, 1)[0]
        assert np.array_equal(orc.decode_culled(s, d)[1], orc.decode_culled(full, d)[1][f0:f0 + c])


def test_parse_rejects_malformed_directory(mc):
    """FORMAT.md §1.2: dir[0] = 0, entries non-decreasing, dir[M] inside the records.  A
    blob whose middle entries decrease or run past dir[M] is refused by mc_parse_header,
    so the host helpers (shards, extract, pipelined host decode) never dereference it."""
    blob = mc.mc_encode(synth.quad_grid(16, 16), 64, 126, 2)
    data = np.array(blob.bytes)
    L = blob.layout
    assert L.num_meshlets >= 4
    mc.parse_header(data)
    dir_off = int(L.off_dir)
    d = data[dir_off:dir_off + 4 * (L.num_meshlets + 1)].view(np.uint32)
    bad = data.copy()
    bad[dir_off:dir_off + 4 * (L.num_meshlets + 1)].view(np.uint32)[2] = d[L.num_meshlets] + 5
    with pytest.raises(mc.MCError, match="not a valid"):
        mc.parse_header(bad)
    bad = data.copy()
    bad[dir_off:dir_off + 4 * (L.num_meshlets + 1)].view(np.uint32)[2] = d[1] - 1
    with pytest.raises(mc.MCError, match="not a valid"):
        mc.parse_header(bad)
    with pytest.raises(mc.MCError):
        mc.mc_blob_shard_ranges(bad, 2)
    with pytest.raises(mc.MCError):
        mc.mc_blob_extract(bad, 0, 2)


def test_object_id_limits(mc):
    """Object ids index the per-object grid table (u16 in the record header, FORMAT.md
    §1.4): ids >= 65536 (including UINT32_MAX, where id + 1 wraps) are MC_ERR_LIMITS."""
    m = synth.quad_grid(4, 4)
    T = m.indices.shape[0]
    for bad_id in (65536, 0xFFFFFFFF):
        obj = np.zeros(T, np.uint32)
        obj[3] = bad_id
        m2 = synth.Mesh(m.indices, m.attributes, m.bits, m.semantic)
        m2.object_of_triangle = obj
        with pytest.raises(mc.MCError, match="limits"):
            mc.mc_encode(m2)
    obj = np.zeros(T, np.uint32)
    obj[T // 2:] = 65535
    m3 = synth.Mesh(m.indices, m.attributes, m.bits, m.semantic)
    m3.object_of_triangle = obj
    b = mc.mc_encode(m3)
    assert b.layout.num_objects == 65536


@pytest.mark.parametrize("codec,vw", [(1, False), (2, False), (3, False), (2, True)])
def test_blob_info_against_oracle_decode(mc, orc, codec, vw):
    """mc_blob_info (P:486-499 grid diagnostics, section sizes) against values computed
    independently: grid extents from the ORACLE's decoded q values and the record fields
    read by tests/streams.py; bit budgets restated from FORMAT.md §1.4."""
    from streams import read_records
    scene = synth.city(num_instances=3, num_prototypes=2, k=10, seed=4)
    protos = [mc.mc_encode(p, 64, 126, codec, variable_widths=vw) for p in scene.prototypes]
    blob = mc.mc_blob_instance(protos, scene.instance_proto, scene.instance_offset)
    data = np.array(blob.bytes)
    info, grids = blob.info()
    L = blob.layout
    err, errs, idx, q, f = orc.decode(data)
    assert err == 0
    recs = read_records(data)
    n, O = L.n, L.num_objects
    qv = q.reshape(-1, n).astype(np.int64)
    lo = np.full((O, n), np.iinfo(np.int64).max)
    hi = np.zeros((O, n), np.int64)
    wmax = np.zeros((O, n), np.int64)
    for r in recs:
        sl = qv[r["vtx_base"]:r["vtx_base"] + r["V"]]
        lo[r["object"]] = np.minimum(lo[r["object"]], sl.min(0))
        hi[r["object"]] = np.maximum(hi[r["object"]], sl.max(0))
        wmax[r["object"]] = np.maximum(wmax[r["object"]], (sl - np.array(r["L"], np.int64)).max(0))
    off_obj = int(L.off_obj)
    tab = data[off_obj:off_obj + 8 * n * O].view(np.float32).reshape(O, 2, n)
    for o in range(O):
        for c in range(n):
            g = grids[o][c]
            assert g["W_steps"] == hi[o, c] - lo[o, c] and g["w_steps"] == wmax[o, c]
            assert g["w_steps"] <= (1 << g["bits"]) - 1          # b bits suffice
            assert g["delta"] == tab[o, 0, c] and g["origin"] == tab[o, 1, c]
            assert g["info_bits"] == (np.log2(g["W_steps"]) if g["W_steps"] else 0.0)
            assert abs(g["W"] - g["W_steps"] * float(tab[o, 0, c])) <= 1e-9 * max(1.0, g["W"])
    # the largest meshlet extent spans the b-bit range (Δ = w/(2^b-1)), non-VW grids
    assert max(grids[o][c]["w_steps"] for o in range(O) for c in range(n)) >= (1 << 16) - 2
    assert info["restarts"] == sum(r["R"] for r in recs)
    assert info["total_t"] == L.total_t and info["num_meshlets"] == len(recs)
    assert (info["header_bytes"] + info["directory_bytes"] + info["object_bytes"] + info["cull_bytes"] +
            info["record_bytes"]) == info["total_bytes"] == data.nbytes
    assert (info["record_header_bytes"] + info["flag_bytes"] + info["index_bytes"] + info["attribute_bytes"] +
            info["padding_bytes"]) == info["record_bytes"]
    W = [0 if codec == 3 else (r["Tp"] + 31) // 32 for r in recs]
    assert info["flag_bytes"] == sum(4 * w * (2 if codec == 2 else 1) for w in W)
    nb = [r["Tp"] - 1 if codec == 1 else 3 * r["Tp"] if codec == 3 else (r["Tp"] - 1) - (r["V"] - 3) for r in recs]
    assert info["index_bytes"] == sum(nb)
    assert info["attribute_bytes"] == sum((r["V"] * sum(r["widths"]) + 7) // 8 for r in recs)
    assert abs(info["bits_per_triangle"] - 8 * data.nbytes / L.total_t) < 1e-9
