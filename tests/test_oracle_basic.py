"""Pins for the oracle's Basic codec (codec 3) and the local u8x4 index output.

Basic is the paper's uncompressed mesh-shading control: "triangles use three indices
stored in the Basic Index Buffer", 8 bits per index, 24 bpt in Table 2
(P:586-591).  The u8x4 output is the same per-meshlet 8-bit index form written as one
u32 per triangle (FORMAT.md §2).  No GPU.  Expected values come from the source meshes,
hand-written streams and the paper's numbers — never from the oracle itself.
"""
import numpy as np
import pytest

import synth
from streams import basic_meshlet, gts_meshlet, pack_meshlets, read_records

CODEC_BASIC = 3


def _src_triangles_from_u8x4(e, words):
    """Map u8x4 words back to source vertices through each record's vertex base."""
    out = []
    for r in read_records(e.blob):
        w = words[r["tri_base"]:r["tri_base"] + r["Tp"]].astype(np.int64)
        loc = np.stack([w & 0xFF, (w >> 8) & 0xFF, (w >> 16) & 0xFF], 1)
        assert np.all((w >> 24) == 0)
        assert np.all(loc < r["V"])
        out.append(e.src_vertex[r["vtx_base"] + loc])
    return np.concatenate(out) if out else np.zeros((0, 3), np.int64)


@pytest.mark.parametrize("mesh", ["grid", "patch3", "patch7", "torus", "sphere", "fan"])
@pytest.mark.parametrize("limits", [(64, 126), (128, 256), (32, 32), (3, 1)])
def test_basic_roundtrip(orc, mesh, limits):
    """Basic decodes to exactly the source triangles, winding preserved, with no
    restarts and no degenerates (T' = T)."""
    m = {"grid": lambda: synth.quad_grid(), "patch3": lambda: synth.random_patch(3),
         "patch7": lambda: synth.random_patch(7), "torus": lambda: synth.torus(30, 16),
         "sphere": lambda: synth.displaced_sphere(9), "fan": lambda: synth.fan(200)}[mesh]()
    e = orc.encode(m, *limits, CODEC_BASIC)
    err, errs, idx, q, f = orc.decode(e.blob)
    assert err == 0
    assert e.stats["restarts"] == 0 and e.stats["total_tp"] == e.stats["total_t"] == len(m.indices)
    tri = idx.reshape(-1, 3).astype(np.int64)
    src = e.src_vertex[tri]
    assert np.array_equal(synth.canonical_triangles(src), synth.canonical_triangles(m.indices))
    assert np.all(e.src_tri != 0xFFFFFFFF)
    for r in read_records(e.blob):
        assert 3 <= r["V"] <= limits[0] and r["Tp"] <= limits[1] and r["R"] == 0


def test_basic_budget_24bpt(orc):
    """P:294 / Table 2: Basic stores 3 x 8 bits per triangle; the record is
    header + 3T' index bytes (padded to 4) + V·S attribute bits, 16-B padded."""
    m = synth.displaced_sphere(12)
    e = orc.encode(m, 64, 126, CODEC_BASIC)
    info = orc.blob_info(e.blob)
    idx_bytes = 0
    for r in read_records(e.blob):
        topo = (3 * r["Tp"] + 3) // 4 * 4
        attr = (r["V"] * info.S + 31) // 32 * 4
        assert r["size"] == (r["hdr"] + topo + attr + 15) // 16 * 16
        idx_bytes += 3 * r["Tp"]
    assert 8 * idx_bytes / len(m.indices) == 24.0


def test_basic_equals_gts_triangle_sets(orc):
    """Basic, GTS and GTS-Reuse encode the same mesh to the same set of real triangles."""
    m = synth.displaced_sphere(8)
    sets = []
    for codec in (1, 2, 3):
        e = orc.encode(m, 64, 126, codec)
        err, errs, idx, q, f = orc.decode(e.blob, want_q=False, want_f=False)
        assert err == 0
        tri = idx.reshape(-1, 3).astype(np.int64)
        deg = (tri[:, 0] == tri[:, 1]) | (tri[:, 1] == tri[:, 2]) | (tri[:, 0] == tri[:, 2])
        sets.append(synth.canonical_triangles(e.src_vertex[tri[~deg]]))
    assert np.array_equal(sets[0], sets[1]) and np.array_equal(sets[0], sets[2])


def test_basic_handwritten_stream(orc):
    """A hand-written Basic record decodes to its own triangle list, including a
    repeated-index triangle passed through as written."""
    tris = [(0, 1, 2), (2, 1, 3), (4, 2, 3), (4, 4, 0)]
    blob = pack_meshlets(orc, CODEC_BASIC, [basic_meshlet(5, tris)])
    err, meta, tri, q, f = orc.decode_meshlet(blob, 0)
    assert err == 0
    assert [tuple(int(x) for x in t) for t in tri] == tris


def test_basic_faults(orc):
    """FORMAT.md §5 for Basic: an index >= V sets INDEX; R != 0 sets COUNTS."""
    bad = pack_meshlets(orc, CODEC_BASIC, [basic_meshlet(3, [(0, 1, 2), (2, 1, 3)])])
    assert orc.decode_meshlet(bad, 0)[0] == orc.DERR_INDEX
    restarts = pack_meshlets(orc, CODEC_BASIC, [basic_meshlet(3, [(0, 1, 2)])], R=[1])
    assert orc.decode_meshlet(restarts, 0)[0] & orc.DERR_COUNTS


@pytest.mark.parametrize("codec", [1, 2, 3])
def test_u8x4_maps_back_to_source(orc, codec):
    """u8x4 words hold meshlet-local indices: through each record's vtx_base and
    the encoder's source map they give back the source triangles (plus 4 degenerates per
    restart for the strip codecs)."""
    m = synth.random_patch(5, nx=20, ny=14)
    e = orc.encode(m, 64, 126, codec)
    err, words = orc.decode_u8x4(e.blob)
    assert err == 0 and words.size == e.stats["total_tp"]
    src = _src_triangles_from_u8x4(e, words)
    deg = (src[:, 0] == src[:, 1]) | (src[:, 1] == src[:, 2]) | (src[:, 0] == src[:, 2])
    assert deg.sum() == 4 * e.stats["restarts"]
    assert np.array_equal(synth.canonical_triangles(src[~deg]), synth.canonical_triangles(m.indices))


def test_u8x4_handwritten_gts(orc):
    """The S:361-style fan stream as u8x4: one word per decoded triangle, local indices."""
    # GTS stream: flags R,L,R (t = 1..3), new vertices 3,4,5 -> sequential walk (FORMAT.md §2)
    blob = pack_meshlets(orc, 1, [gts_meshlet(6, [1, 0, 1], [3, 4, 5])])
    err, words = orc.decode_u8x4(blob)
    assert err == 0
    want = [(0, 1, 2), (2, 1, 3), (2, 3, 4), (4, 3, 5)]
    assert [(int(w) & 255, (int(w) >> 8) & 255, (int(w) >> 16) & 255) for w in words] == want
