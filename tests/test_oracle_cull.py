"""Pins for cone-culled, compacted decode (FORMAT.md §1.5, §7).

The paper culls whole meshlets in the amplification shader when a normal cone shows
every triangle back-facing, which it reports as worth up to 1.6x.
The oracle's culled decode (or_decode_culled) is pinned here against the already-pinned
full decode plus a prefix sum restated from FORMAT.md §7, against hand-set cull tables
(never / always / chosen subsets / the exact decision boundary), and — for cones the
product encoder computes — by brute force: a culled meshlet's real triangles must all be
back-facing in double precision.  No GPU.
"""
import numpy as np
import pytest

import synth
from streams import read_records


def _full(orc, blob):
    err, errs, idx, q, f = orc.decode(blob)
    assert err == 0
    return idx, q, f


def _expected_compacted(orc, blob, visible):
    """FORMAT.md §7 restated: visible records in record order, output bases = exclusive
    prefix sums of V and T' over the visible ones."""
    info = orc.blob_info(blob)
    idx, q, f = _full(orc, blob)
    recs = read_records(blob)
    ei, eq, ef = [], [], []
    VB = 0
    for r, v in zip(recs, visible):
        if not v:
            continue
        t = idx[3 * r["tri_base"]:3 * (r["tri_base"] + r["Tp"])].astype(np.int64) - r["vtx_base"] + VB
        ei.append(t.astype(np.uint32))
        eq.append(q[info.n * r["vtx_base"]:info.n * (r["vtx_base"] + r["V"])])
        ef.append(f[info.n_out * r["vtx_base"]:info.n_out * (r["vtx_base"] + r["V"])])
        VB += r["V"]
    cat = lambda xs, dt: np.concatenate(xs) if xs else np.zeros(0, dt)
    return cat(ei, np.uint32), cat(eq, np.uint32), cat(ef, np.float32)


def _blob(orc, codec=2):
    return orc.encode(synth.displaced_sphere(14), 64, 126, codec).blob


@pytest.mark.parametrize("codec", [1, 2, 3])
def test_cull_never_and_always(orc, codec):
    blob = _blob(orc, codec)
    M = orc.blob_info(blob).M
    never = orc.add_cull(blob, np.tile([0, 0, 1, 2.0], (M, 1)))
    err, vis, c, idx, q, f = orc.decode_culled(never, [0, 0, 1])
    fi, fq, ff = _full(orc, blob)
    assert err == 0 and vis.all() and c["records"] == M
    assert np.array_equal(idx, fi) and np.array_equal(q, fq) and np.array_equal(f.view(np.uint32), ff.view(np.uint32))
    always = orc.add_cull(blob, np.tile([0, 0, 1, -2.0], (M, 1)))
    err, vis, c, idx, q, f = orc.decode_culled(always, [0.3, -0.2, 0.9])
    assert err == 0 and not vis.any() and c == {"records": 0, "V": 0, "Tp": 0, "T": 0} and idx.size == 0


@pytest.mark.parametrize("seed", range(4))
def test_cull_subset_compaction(orc, seed):
    """A chosen subset is culled (axis = d, cutoff 0.5); the rest (cutoff 2) decode into
    compacted buffers exactly as FORMAT.md §7 states."""
    blob = _blob(orc, 2 if seed % 2 else 1)
    M = orc.blob_info(blob).M
    rng = np.random.default_rng(seed)
    d = rng.normal(size=3).astype(np.float32)
    d /= np.linalg.norm(d)
    cull = rng.random(M) < 0.45
    ent = np.zeros((M, 4), np.float32)
    ent[:, :3] = d
    ent[:, 3] = np.where(cull, 0.5, 2.0)
    cb = orc.add_cull(blob, ent)
    err, vis, c, idx, q, f = orc.decode_culled(cb, d)
    assert err == 0 and np.array_equal(vis, ~cull)
    ei, eq, ef = _expected_compacted(orc, blob, ~cull)
    assert np.array_equal(idx, ei) and np.array_equal(q, eq) and np.array_equal(f.view(np.uint32), ef.view(np.uint32))
    recs = read_records(blob)
    assert c["V"] == sum(r["V"] for r, v in zip(recs, ~cull) if v)
    assert c["Tp"] == sum(r["Tp"] for r, v in zip(recs, ~cull) if v)
    # u8x4 words of the visible records, compacted (FORMAT.md §2, §7)
    err, vis, c8, w8, _, _ = orc.decode_culled(cb, d, u8x4=True, want_q=False, want_f=False)
    _, full8 = orc.decode_u8x4(blob)
    exp8 = np.concatenate([full8[r["tri_base"]:r["tri_base"] + r["Tp"]] for r, v in zip(recs, ~cull) if v])
    assert np.array_equal(w8, exp8)


def test_cull_decision_boundary(orc):
    """The decision is a strict binary32 comparison of fmaf(az,dz,fmaf(ay,dy,ax*dx))."""
    blob = _blob(orc)
    M = orc.blob_info(blob).M
    ent = np.zeros((M, 4), np.float32)
    ent[:, 0] = 1.0
    ent[0::2, 3] = 1.0                                           # s == cutoff: visible
    ent[1::2, 3] = np.nextafter(np.float32(1.0), np.float32(0))  # s > cutoff: culled
    err, vis, c, *_ = orc.decode_culled(orc.add_cull(blob, ent), [1, 0, 0])
    assert np.array_equal(vis, np.arange(M) % 2 == 0)


def test_cull_table_replaced_and_header(orc):
    blob = _blob(orc)
    M = orc.blob_info(blob).M
    a = orc.add_cull(blob, np.tile([0, 0, 1, 2.0], (M, 1)))
    b = orc.add_cull(a, np.tile([0, 0, 1, -2.0], (M, 1)))       # replace, not append
    assert b.nbytes == a.nbytes and int(b[60]) & 2
    assert not orc.decode_culled(b, [0, 0, 1])[1].any()
    # the full decode ignores the cull table
    assert np.array_equal(orc.decode(b)[2], orc.decode(blob)[2])
