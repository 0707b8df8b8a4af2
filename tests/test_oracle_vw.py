"""Pins for per-meshlet attribute widths (FORMAT.md §1.4 `VW`).

The paper quantises every channel to b bits on a crack-free global grid
and notes the information content per channel is fractional (13.4/13.4/13.9 bits for
Rock positions at LW's precision).  `VW` keeps the global grid and stores,
per meshlet and channel, only w_c = bit length of the meshlet's largest code.  Because
the grid is unchanged, a VW blob must decode to exactly the fixed-width blob's values.
No GPU; expected values come from the fixed-width oracle path, the decoded data
(brute force over each meshlet) and FORMAT.md's size rule.
"""
import numpy as np
import pytest

import synth
from streams import read_records

MESHES = {
    "grid": lambda: synth.quad_grid(),
    "sphere_oct": lambda: synth.displaced_sphere(14),
    "sphere_nrm10": lambda: synth.displaced_sphere(14, oct_normals=False).with_bits(10),
    "patch_mixed": lambda: synth.random_patch(4),
    "torus24": lambda: synth.torus(40, 20).with_bits(24),
}


@pytest.mark.parametrize("name", list(MESHES))
@pytest.mark.parametrize("codec", [1, 2, 3])
def test_vw_decodes_like_fixed(orc, name, codec):
    m = MESHES[name]()
    fixed = orc.encode(m, 64, 126, codec)
    var = orc.encode(m, 64, 126, codec, vw=True)
    a = orc.decode(fixed.blob)
    b = orc.decode(var.blob)
    assert a[0] == 0 and b[0] == 0
    assert np.array_equal(a[2], b[2])                          # indices
    assert np.array_equal(a[3], b[3])                          # q on the global grid
    assert np.array_equal(a[4].view(np.uint32), b[4].view(np.uint32))   # floats, bit for bit
    assert orc.blob_info(var.blob).vw == 1 and orc.blob_info(fixed.blob).vw == 0


@pytest.mark.parametrize("name", list(MESHES))
def test_vw_width_is_bit_length_of_largest_code(orc, name):
    """Brute force per meshlet: codes = q - L_c from the decode; every code < 2^w_c and
    the largest code has bit length exactly w_c (w_c = 0 iff all codes are 0)."""
    m = MESHES[name]()
    e = orc.encode(m, 64, 126, 2, vw=True)
    info = orc.blob_info(e.blob)
    err, errs, idx, q, f = orc.decode(e.blob)
    assert err == 0
    q = q.reshape(-1, info.n).astype(np.int64)
    for r in read_records(e.blob):
        codes = q[r["vtx_base"]:r["vtx_base"] + r["V"]] - np.array(r["L"], np.int64)
        assert codes.min() >= 0
        for c in range(info.n):
            w, mx = r["widths"][c], int(codes[:, c].max())
            assert mx < (1 << w) and mx.bit_length() == w
            assert w <= m.bits[c]


def test_vw_record_size_rule(orc):
    m = MESHES["sphere_oct"]()
    for codec in (1, 2, 3):
        e = orc.encode(m, 64, 126, codec, vw=True)
        n = orc.blob_info(e.blob).n
        for r in read_records(e.blob):
            V, Tp = r["V"], r["Tp"]
            W = 0 if codec == 3 else (Tp + 31) // 32
            nb = {1: Tp - 1, 2: (Tp - 1) - (V - 3), 3: 3 * Tp}[codec]
            topo = 4 * W * (2 if codec == 2 else 1) + (nb + 3) // 4 * 4
            attr = (V * sum(r["widths"]) + 31) // 32 * 4
            assert r["hdr"] == (16 + 5 * n + 15) // 16 * 16
            assert r["size"] == (r["hdr"] + topo + attr + 15) // 16 * 16


def test_vw_saves_bits_on_smooth_surfaces(orc):
    """Meshlets cover a small part of a smooth surface, so position codes need fewer
    than the global 16 bits (the paper's observation behind P:715-716)."""
    m = synth.displaced_sphere(24)
    e = orc.encode(m, 64, 126, 2, vw=True)
    ws = np.array([r["widths"] for r in read_records(e.blob)])
    assert ws[:, :3].mean() < 15.0 and ws[:, 3:5].mean() < 14.0   # positions, oct normals
    fixed = orc.encode(m, 64, 126, 2)
    assert e.blob.nbytes < 0.98 * fixed.blob.nbytes


def test_vw_faults(orc):
    """A record width above the blob's b_c is a RECORD error (FORMAT.md §5); an unknown
    header flag bit is not a FORMAT.md blob."""
    e = orc.encode(MESHES["grid"](), 64, 126, 2, vw=True)
    blob = e.blob.copy()
    r = read_records(blob)[1]
    n = orc.blob_info(blob).n
    blob[r["offset"] + 16 + 4 * n] = 17                        # b_0 = 16
    err, errs, idx, q, f = orc.decode(blob)
    assert errs[1] == orc.DERR_RECORD and errs[0] == 0
    bad = e.blob.copy()
    bad[60] |= 4
    with pytest.raises(ValueError):
        orc.blob_info(bad)
