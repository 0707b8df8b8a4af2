"""Pins for the oracle (oracle/oracle.c) against what the paper and mathematics fix.

No GPU.  Each test names the passage it pins.  Expected values come from the
paper/SPEC text (tests/golden/paper_examples.json), from the synthetic source mesh
(round trips), from closed forms, or from brute force — never from the oracle itself
and never from the CUDA path.
"""
import itertools
import json
import os

import numpy as np
import pytest

import synth
from streams import (closed_form_decode, gts_meshlet, pack_meshlets, py_strip_encode, read_records,
                     reuse_fields, reuse_meshlet)

pytestmark = pytest.mark.filterwarnings("ignore")
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")))
FL = {"R": 1, "L": 0}


def _tris(orc, blob, m=0):
    err, meta, tri, q, f = orc.decode_meshlet(blob, m)
    return err, [tuple(int(x) for x in t) for t in tri]


# ------------------------------------------------------------------ worked examples

@pytest.mark.parametrize("ex", GOLD["sequential_decode"], ids=lambda e: e["cite"])
def test_spec_sequential_examples(orc, ex):
    flags = [FL[f] for f in ex["flags"]]
    if ex["codec"] == "gts":
        blob = pack_meshlets(orc, 1, [gts_meshlet(ex["V"], flags, ex["idx"])])
        err, tris = _tris(orc, blob)
        assert err == 0
        assert tris == [tuple(t) for t in ex["expect_tris"]]
    else:
        blob = pack_meshlets(orc, 2, [reuse_meshlet(ex["V"], flags, ex["inc"], ex["reuse"])])
        err, tris = _tris(orc, blob)
        assert err == 0
        assert [t[2] for t in tris[1:]] == ex["expect_new_vertex_sequence"]


def test_restart_pattern_S353(orc):
    """Relabel S:353's example onto locals: (a,b,c)=(0,1,2) plays (3,7,9), q,p,r = 3,4,5."""
    g = GOLD["restart"]
    lab = {g["prev"][0]: 0, g["prev"][1]: 1, g["prev"][2]: 2, g["q"]: 3, g["p"]: 4, g["r"]: 5}
    c, q, p, r = 2, 3, 4, 5
    blob = pack_meshlets(orc, 1, [gts_meshlet(6, [1, 0, 0, 1, 1], [c, q, q, p, r])], R=[1])
    err, tris = _tris(orc, blob)
    assert err == 0
    assert tris[1:5] == [tuple(lab[v] for v in t) for t in g["expect_degenerates"]]
    assert tris[5] == tuple(lab[v] for v in g["expect_real"])
    assert all(len(set(t)) < 3 for t in tris[1:5])


def test_lookback_example_S442():
    g = GOLD["lookback"]
    f = [0] + [FL[x] for x in g["flags_from_t1"]]
    t = g["t"]
    j = max(k for k in range(t) if f[k] != f[t])
    assert j == g["expect_j"]


def test_fan_encode_S335(orc):
    """Encoding a 3-triangle fan gives flags [L,L], indices [3,4], increment flags [1,1]."""
    g = GOLD["fan_encode"]
    V, flags, N, src = py_strip_encode([tuple(t) for t in g["fan"]], [[0, 1, 2]])
    # the fan's first triangle must be rotated so its successor is reachable; relabelled
    # locals then follow first appearance
    assert [("R" if f else "L") for f in flags] == g["expect_flags"]
    assert N[3:] == g["expect_idx"]
    inc, reuse = reuse_fields(N)
    assert inc == g["expect_inc"] and reuse == []
    m = synth.fan(3)
    e = orc.encode(m, 64, 126, orc.CODEC_GTS)
    rec = read_records(e.blob)[0]
    assert rec["Tp"] == 3 and rec["V"] == 5
    err, tris = _tris(orc, e.blob)
    assert err == 0 and len(tris) == 3


def test_paper_fan_statement_P435(orc):
    """Partial pin (Fig. 2 is missing): 'triangle 8 requires the index of triangle 4, which
    is 0'.  A stream whose triangle 4 re-uses vertex 0 and whose triangles 6..8 share a flag
    that differs from triangle 5's must hand vertex 0 to triangle 8 (lookback j(8)=5 -> N[6])."""
    flags = [1, 1, 0, 1, 0, 1, 1, 1]            # f_1..f_8; f_5 = L, f_6..8 = R
    idx = [3, 4, 5, 0, 6, 7, 8, 9]              # triangle 4's index is vertex 0
    blob = pack_meshlets(orc, 1, [gts_meshlet(10, flags, idx)])
    err, tris = _tris(orc, blob)
    assert err == 0
    assert tris[8][1] == 0 and tris[4][2] == 0


def test_table1_degenerates_are_4x_restarts():
    for row in GOLD["table1_restarts"]["rows"]:
        assert row["degenerates"] == 4 * row["restarts"]


# ------------------------------------------------------------------ closed form == sequential (V1)

def test_closed_form_exhaustive_16(orc):
    """All 2^15 L/R patterns of T'=16: sequential oracle == independently written
    closed-form lookback."""
    Tp = 16
    pats = list(itertools.product([0, 1], repeat=Tp - 1))
    idx = list(range(3, Tp + 2))
    blob = pack_meshlets(orc, 1, [gts_meshlet(Tp + 2, p, idx) for p in pats])
    err, errs, out, q, f = orc.decode(blob, want_q=False, want_f=False)
    assert err == 0
    got = out.reshape(len(pats), Tp, 3).astype(np.int64) - (np.arange(len(pats)) * (Tp + 2))[:, None, None]
    N = [0, 1, 2] + idx
    for i in range(0, len(pats), 97):  # python closed form is slow; stride-sample + full check below
        assert [tuple(t) for t in got[i]] == closed_form_decode(pats[i], N)
    # full check, vectorised closed form
    F = np.concatenate([np.zeros((len(pats), 1), np.int64), np.array(pats)], 1)
    Na = np.array(N)
    for t in range(1, Tp):
        diff = F[:, :t] != F[:, t:t + 1]
        has = diff.any(1)
        j = np.where(has, t - 1 - np.argmax(diff[:, ::-1], 1), -1)
        pj = Na[j + 1]
        exp0 = np.where(F[:, t] == 1, Na[t + 1], pj)
        exp1 = np.where(F[:, t] == 1, pj, Na[t + 1])
        assert np.array_equal(got[:, t, 0], exp0)
        assert np.array_equal(got[:, t, 1], exp1)
        assert np.all(got[:, t, 2] == Na[t + 2])


def test_closed_form_long_fans(orc):
    """Random T'=256 patterns with long same-flag runs crossing several 32-bit words."""
    rng = np.random.default_rng(1)
    ms, pats = [], []
    for k in range(60):
        Tp = int(rng.integers(33, 257))
        f, cur = [], int(rng.integers(0, 2))
        while len(f) < Tp - 1:
            run = int(rng.integers(1, 90))
            f += [cur] * run
            cur ^= 1
        f = f[:Tp - 1]
        idx = list(rng.integers(0, 256, size=Tp - 1))
        ms.append(gts_meshlet(256, f, idx))
        pats.append((f, [0, 1, 2] + [int(x) for x in idx]))
    blob = pack_meshlets(orc, 1, ms)
    for m, (f, N) in enumerate(pats):
        err, tris = _tris(orc, blob, m)
        assert err == 0
        assert tris == closed_form_decode(f, N)


# ------------------------------------------------------------------ brute force over path covers

def _path_covers(tris, adj):
    """Every ordered path cover of a tiny meshlet (all orderings / directions of paths)."""
    n = len(tris)

    def paths_from(start, used):
        yield [start]
        for nb in adj[start]:
            if nb not in used:
                for rest in paths_from(nb, used | {nb}):
                    yield [start] + rest

    def covers(remaining):
        if not remaining:
            yield []
            return
        for s in sorted(remaining):
            for p in paths_from(s, frozenset([s])):
                if set(p) <= remaining:
                    for rest in covers(remaining - set(p)):
                        yield [p] + rest

    yield from covers(frozenset(range(n)))


def _adjacency(tris):
    adj = {i: [] for i in range(len(tris))}
    for i, j in itertools.combinations(range(len(tris)), 2):
        ei = {(tris[i][k], tris[i][(k + 1) % 3]) for k in range(3)}
        ej = {(tris[j][(k + 1) % 3], tris[j][k]) for k in range(3)}
        if ei & ej:
            adj[i].append(j)
            adj[j].append(i)
    return adj


@pytest.mark.parametrize("mesh_id", range(7))
def test_bruteforce_path_covers_roundtrip(orc, mesh_id):
    """Every path cover (all path orders and directions) of tiny patches of 4-6 triangles
    (SURVEY §8(c) "meshlets of <= 6 triangles"), encoded by an independent Python encoder,
    decodes (GTS and Reuse) to the source triangles with winding preserved."""
    grid = synth.quad_grid(3, 2).indices
    picks = [[0, 1, 2, 3], [0, 1, 2, 3, 4], [1, 2, 3, 4, 5], [2, 3, 6, 7, 8],
             [0, 1, 2, 3, 4, 5], [2, 3, 4, 5, 6, 7], [0, 1, 2, 3, 6, 7]][mesh_id]
    tris = [tuple(int(v) for v in grid[p]) for p in picks]
    adj = _adjacency(tris)
    covers = list(_path_covers(tris, adj))
    assert 3 < len(covers) <= 4000          # every cover is checked
    gts, reu, srcs = [], [], []
    for cov in covers:
        V, flags, N, src = py_strip_encode(tris, cov)
        gts.append(gts_meshlet(V, flags, N[3:]))
        inc, reuse = reuse_fields(N)
        reu.append(reuse_meshlet(V, flags, inc, reuse))
        srcs.append((src, len(cov) - 1))
    want = synth.canonical_triangles(np.array(tris))
    for codec, ms in ((1, gts), (2, reu)):
        blob = pack_meshlets(orc, codec, ms, R=[r for _, r in srcs])
        err, errs, idx, q, f = orc.decode(blob, want_q=False, want_f=False)
        assert err == 0
        recs = read_records(blob)
        for m, (src, R) in enumerate(srcs):
            r = recs[m]
            t = idx[3 * r["tri_base"]:3 * (r["tri_base"] + r["Tp"])].reshape(-1, 3) - r["vtx_base"]
            g = np.array(src)[t]
            real = g[(g[:, 0] != g[:, 1]) & (g[:, 1] != g[:, 2]) & (g[:, 0] != g[:, 2])]
            assert r["Tp"] == len(tris) + 4 * R
            assert np.array_equal(synth.canonical_triangles(real), want)


# ------------------------------------------------------------------ round trips on scenes

def _roundtrip(orc, mesh, vmax, tmax, codec):
    e = orc.encode(mesh, vmax, tmax, codec)
    err, errs, idx, q, f = orc.decode(e.blob)
    assert err == 0
    tri = idx.reshape(-1, 3).astype(np.int64)
    src = e.src_vertex[tri]
    deg = (tri[:, 0] == tri[:, 1]) | (tri[:, 1] == tri[:, 2]) | (tri[:, 0] == tri[:, 2])
    # every restart contributes exactly four degenerates (Table 1)
    assert deg.sum() == 4 * e.stats["restarts"]
    assert e.stats["total_tp"] == e.stats["total_t"] + 4 * e.stats["restarts"]
    # winding-preserving round trip of the triangle multiset
    assert np.array_equal(synth.canonical_triangles(src[~deg]), synth.canonical_triangles(mesh.indices))
    # real (non-degenerate) slots map back to their source triangles
    st = e.src_tri
    assert np.all((st == 0xFFFFFFFF) == deg)
    return e, idx, q, f


@pytest.mark.parametrize("codec", [1, 2])
@pytest.mark.parametrize("limits", [(64, 126), (128, 256), (32, 32), (256, 256), (3, 1), (16, 8)])
def test_roundtrip_grid(orc, codec, limits):
    e, idx, q, f = _roundtrip(orc, synth.quad_grid(), *limits, codec)
    for r in read_records(e.blob):
        assert 3 <= r["V"] <= limits[0] and r["Tp"] <= limits[1]


@pytest.mark.parametrize("seed", range(12))
def test_roundtrip_random_patches(orc, seed):
    m = synth.random_patch(seed)
    for codec in (1, 2):
        _roundtrip(orc, m, [64, 32, 128][seed % 3], [126, 64, 256][seed % 3], codec)


def test_roundtrip_surfaces(orc):
    for m in (synth.torus(40, 20), synth.displaced_sphere(12), synth.fan(255), synth.fan(40)):
        for codec in (1, 2):
            _roundtrip(orc, m, 64, 126, codec)


def test_gts_and_reuse_decode_identically(orc):
    """both codecs decode a meshlet to identical triangle lists."""
    m = synth.displaced_sphere(10)
    a = orc.decode(orc.encode(m, 64, 126, 1).blob)
    b = orc.decode(orc.encode(m, 64, 126, 2).blob)
    assert np.array_equal(a[2], b[2]) and np.array_equal(a[3], b[3])
    assert np.array_equal(a[4].view(np.uint32), b[4].view(np.uint32))


def test_reuse_invariants(orc):
    """#increment flags = V-3, reuse length = (T'-1)-(V-3); the paper's reuse
    location t+1-s equals reuse[t - c_t - 1] with s = 2 + c_t (reading R5), checked
    against step sequences recovered from the decoded triangles."""
    m = synth.random_patch(5)
    e = orc.encode(m, 64, 126, 2)
    err, errs, idx, q, f = orc.decode(e.blob, want_q=False, want_f=False)
    b = e.blob
    for r in read_records(b):
        V, Tp = r["V"], r["Tp"]
        pc = sum(bin(int(w)).count("1") for w in r["inc"])
        assert pc == V - 3
        nbytes = (Tp - 1) - (V - 3)
        W = (Tp + 31) // 32
        off = r["offset"] + r["hdr"] + 8 * W
        reuse = list(b[off:off + nbytes])
        tri = idx[3 * r["tri_base"]:3 * (r["tri_base"] + Tp)].reshape(-1, 3) - r["vtx_base"]
        N = [0, 1, 2] + [int(t[2]) for t in tri[1:]]
        incs = [(int(r["inc"][t // 32]) >> (t % 32)) & 1 for t in range(Tp)]
        s = 2
        for t in range(1, Tp):
            if incs[t]:
                s += 1
                assert N[t + 2] == s                       # "flag 1: s is the current index"
            else:
                assert N[t + 2] == reuse[(t + 1 - s)]      # "reuse array at location t+1-s"


# ------------------------------------------------------------------ quantisation

def _q_check(orc, mesh, e, q, f):
    info = orc.blob_info(e.blob)
    n = info.n
    qv = q.reshape(-1, n).astype(np.int64)
    A = mesh.attributes[e.src_vertex].astype(np.longdouble)
    recs = read_records(e.blob)
    off_obj = int(np.frombuffer(e.blob[72:80].tobytes(), "<u8")[0])
    O = info.O
    tab = np.frombuffer(e.blob[off_obj:off_obj + 8 * n * O].tobytes(), "<f4").reshape(O, 2, n)
    for r in recs:
        sl = slice(r["vtx_base"], r["vtx_base"] + r["V"])
        d = tab[r["object"], 0].astype(np.longdouble)
        g = tab[r["object"], 1].astype(np.longdouble)
        # error <= Δ/2 in (80-bit) exact arithmetic: q*Δ has <= 56 significant bits
        recon = g + qv[sl].astype(np.longdouble) * d
        assert np.all(np.abs(A[sl] - recon) <= d / 2 * (1 + 1e-9))
        # codes relative to L fit b bits, and L is the meshlet minimum
        codes = qv[sl] - np.array(r["L"], np.int64)
        assert np.all(codes >= 0)
        assert np.all(codes.max(0) <= (1 << np.array(mesh.bits, np.int64)) - 1)
        assert np.all(codes.min(0) == 0)
    return tab


@pytest.mark.parametrize("bits", [8, 10, 12, 16, 20, 24])
def test_quantization_error_and_fit(orc, bits):
    m = synth.quad_grid(16, 16, bits=bits)
    e = orc.encode(m, 64, 126, 2)
    err, errs, idx, q, f = orc.decode(e.blob)
    _q_check(orc, m, e, q, f)


def test_quantization_random_widths(orc):
    for seed in range(6):
        m = synth.random_patch(seed + 100)
        e = orc.encode(m, 32, 64, 2)
        err, errs, idx, q, f = orc.decode(e.blob)
        _q_check(orc, m, e, q, f)


def test_crack_free(orc):
    """Duplicated boundary vertices decode bit-identically in every meshlet."""
    m = synth.displaced_sphere(14, oct_normals=True)
    e = orc.encode(m, 64, 126, 2)
    err, errs, idx, q, f = orc.decode(e.blob)
    info = orc.blob_info(e.blob)
    qv = q.reshape(-1, info.n)
    fv = f.view(np.uint32).reshape(-1, info.n_out)
    order = np.argsort(e.src_vertex, kind="stable")
    sv = e.src_vertex[order]
    dup = np.nonzero(sv[1:] == sv[:-1])[0]
    assert dup.size > 100
    assert np.array_equal(qv[order][dup], qv[order][dup + 1])
    assert np.array_equal(fv[order][dup], fv[order][dup + 1])


def test_quantization_example_S518(orc):
    """S:518 scaled by 65535 so Δ = w/(2^b-1) = 1 exactly: {0, 32767.5, 65535} -> {0, 32768, 65535}
    (round half up, origin at the minimum)."""
    g = GOLD["quantization"]
    pos = np.array([[g["values"][0], 0, 0], [g["values"][1], 1, 0], [g["values"][2], 0, 1]], np.float32)
    mesh = synth.Mesh(np.array([[0, 1, 2]], np.uint32), pos[:, :1].copy(), [g["bits"]], [0])
    e = orc.encode(mesh, 64, 126, 2)
    err, meta, tri, q, f = orc.decode_meshlet(e.blob, 0)
    codes = q[:, 0] - q[:, 0].min()
    got = {int(e.src_vertex[i]): int(codes[i]) for i in range(3)}
    assert [got[0], got[1], got[2]] == g["expect_codes"]
    tab = np.frombuffer(e.blob[int(np.frombuffer(e.blob[72:80].tobytes(), "<u8")[0]):][:8].tobytes(), "<f4")
    assert tab[0] == 1.0  # Δ = 65535 / (2^16 - 1)


def test_constant_channel(orc):
    """a constant channel gets all-zero codes and decodes exactly."""
    m = synth.quad_grid(4, 4)
    attr = m.attributes.copy()
    attr[:, 2] = 5.0
    m2 = synth.Mesh(m.indices, attr, m.bits, m.semantic)
    e = orc.encode(m2, 64, 126, 2)
    err, errs, idx, q, f = orc.decode(e.blob)
    fv = f.reshape(-1, 8)
    assert np.all(fv[:, 2] == 5.0)
    for r in read_records(e.blob):
        qv = q.reshape(-1, 8)[r["vtx_base"]:r["vtx_base"] + r["V"], 2]
        assert np.all(qv == r["L"][2])


def test_information_content(orc):
    """log2(W_i/Δ_i) >= b per channel (>= b - 0.01 allowing the fp32 Δ)."""
    m = synth.torus(60, 30)
    e = orc.encode(m, 64, 126, 2)
    off_obj = int(np.frombuffer(e.blob[72:80].tobytes(), "<u8")[0])
    d = np.frombuffer(e.blob[off_obj:off_obj + 12].tobytes(), "<f4")
    A = m.attributes.astype(np.float64)
    W = A.max(0) - A.min(0)
    info = np.log2(W / d)
    assert np.all(info >= 16 - 0.01)
    assert np.any(info > 16.5)  # many meshlets: global extent > meshlet extent (Table 3)


# ------------------------------------------------------------------ octahedral (extension; closed forms)

def test_oct_special_cases(orc):
    cases = {(0.0, 0.0): (0, 0, 1), (1.0, 0.0): (1, 0, 0), (0.0, 1.0): (0, 1, 0), (-1.0, 0.0): (-1, 0, 0),
             (0.0, -1.0): (0, -1, 0), (1.0, 1.0): (0, 0, -1), (-1.0, -1.0): (0, 0, -1)}
    for (x, y), want in cases.items():
        got = orc.oct_decode(x, y)
        assert np.array_equal(np.abs(got - np.array(want, np.float32)) == 0, np.ones(3, bool)), (x, y, got)


def test_oct_inverse_of_encode(orc):
    rng = np.random.default_rng(3)
    v = rng.normal(size=(2000, 3))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    e = synth.oct_encode(v).astype(np.float32)
    out = np.array([orc.oct_decode(float(a), float(b)) for a, b in e])
    assert np.abs(out - v).max() < 2e-6
    assert np.abs(np.linalg.norm(out.astype(np.float64), axis=1) - 1).max() < 3e-7


def _oct_inputs():
    """(ex, ey) pairs: uniform on [-1,1]^2, both octahedron halves, the 16-bit grid of
    FORMAT.md §3 (q·Δ + g with Δ = 2/(2^16-1), g = -1), fold boundaries and tiny values."""
    rng = np.random.default_rng(5)
    u = rng.uniform(-1, 1, size=(20000, 2))
    d, g = np.float32(2.0 / 65535.0), np.float32(-1.0)
    qg = rng.integers(0, 65536, size=(20000, 2)).astype(np.float32)
    grid = (qg * np.float64(d) + np.float64(g))            # values near the grid, any rounding
    edge = np.array([[a, b] for a in (-1, -0.5, -1e-30, 0.0, 1e-30, 0.5, 1) for b in (-1, -0.75, 0.0, 0.25, 1)])
    diag = np.stack([np.linspace(-1, 1, 4001), 1 - np.abs(np.linspace(-1, 1, 4001))], 1)   # z = 0 fold line
    return np.concatenate([u, grid, edge, diag, -diag]).astype(np.float32)


def test_oct_vs_float64_normalisation(orc):
    """FORMAT.md §4.3 (R13) against float64 (no pin from the paper: the paper only cites
    octahedral normals).  Error analysis of the binary32 sequence (u = 2^-24):
    the fold rounds x, y once and z twice (absolute <= u each, values <= 1); the folded
    vector has |v| >= 1/sqrt(3) (|x|+|y|+|z| = 1), so normalising amplifies that by
    <= sqrt(3) (<= 2.1u); s2 (3 roundings incl. x*x) <= 2u relative, sqrt u, reciprocal u,
    product u -> <= 4u relative on each component.  Bound: |n32 - n64| <= 2^-21 (= 8u)
    absolute per component, where n64 = normalize(fold(ex, ey)) in float64."""
    e = _oct_inputs()
    out = np.array([orc.oct_decode(float(a), float(b)) for a, b in e], np.float64)
    ex, ey = e[:, 0].astype(np.float64), e[:, 1].astype(np.float64)
    z = 1 - np.abs(ex) - np.abs(ey)
    sx, sy = np.where(ex >= 0, 1.0, -1.0), np.where(ey >= 0, 1.0, -1.0)
    x = np.where(z < 0, (1 - np.abs(ey)) * sx, ex)
    y = np.where(z < 0, (1 - np.abs(ex)) * sy, ey)
    v = np.stack([x, y, z], 1)
    n64 = v / np.linalg.norm(v, axis=1, keepdims=True)
    err = np.abs(out - n64)
    assert err.max() <= 2.0 ** -21, err.max()
    # the fold branch is taken (z < 0) for a good share of the inputs, and z = 0 exactly on the diagonals
    assert (z < 0).mean() > 0.3


def test_oct_normalisation_ulp_bound(orc):
    """The normalisation step alone: with the fold evaluated in binary32 (numpy float32
    arithmetic is IEEE RN), each output component is within 4 ulp (binary32) of the
    float64 quotient c / |v| of the same folded vector (the <= 4u relative bound above)."""
    e = _oct_inputs()
    out = np.array([orc.oct_decode(float(a), float(b)) for a, b in e], np.float32)
    one = np.float32(1)
    ex, ey = e[:, 0], e[:, 1]
    ax, ay = np.abs(ex), np.abs(ey)
    z = (one - ax) - ay
    x = np.where(z < 0, (one - ay) * np.where(ex >= 0, one, -one), ex).astype(np.float32)
    y = np.where(z < 0, (one - ax) * np.where(ey >= 0, one, -one), ey).astype(np.float32)
    v = np.stack([x, y, z], 1).astype(np.float64)
    q = v / np.linalg.norm(v, axis=1, keepdims=True)
    ulp = np.spacing(np.abs(q).astype(np.float32)).astype(np.float64)
    nz = q != 0
    ulps = np.abs(out.astype(np.float64) - q)[nz] / ulp[nz]
    assert ulps.max() <= 4.0, ulps.max()
    assert np.all(out[~nz] == 0)          # exact zeros stay zero (x, y or z = 0)


# ------------------------------------------------------------------ budgets

def test_bit_budgets(orc):
    g = GOLD["budgets"]
    assert 3 * 32 == g["vertex_pipeline_bpt"] and 3 * 8 == g["basic_bpt"]
    assert round((8 * 255 + 256) / 256, 2) == g["gts_256_bpt"]
    m = synth.displaced_sphere(12)
    for codec in (1, 2):
        e = orc.encode(m, 64, 126, codec)
        info = orc.blob_info(e.blob)
        for r in read_records(e.blob):
            V, Tp = r["V"], r["Tp"]
            W = (Tp + 31) // 32
            nb = Tp - 1 if codec == 1 else (Tp - 1) - (V - 3)
            topo = 4 * W * (2 if codec == 2 else 1) + (nb + 3) // 4 * 4
            attr = (V * info.S + 31) // 32 * 4
            assert r["size"] == (r["hdr"] + topo + attr + 15) // 16 * 16


# ------------------------------------------------------------------ fault injection

def test_fault_injection(orc):
    m = synth.quad_grid(8, 8)
    e = orc.encode(m, 32, 48, 2)
    recs = read_records(e.blob)
    base = orc.decode(e.blob)[2]
    # flip an increment flag -> popcount != V-3 -> COUNTS error on that meshlet only
    b = e.blob.copy()
    k = 3
    r = recs[k]
    off = r["offset"] + r["hdr"] + 4 * ((r["Tp"] + 31) // 32)
    b[off] ^= 0x02
    err, errs, idx, q, f = orc.decode(b)
    assert errs[k] & orc.DERR_COUNTS and np.count_nonzero(errs) == 1
    # flip an L/R flag -> no format error, but exactly that meshlet's triangles change
    b = e.blob.copy()
    b[r["offset"] + r["hdr"]] ^= 0x04
    err, errs, idx, q, f = orc.decode(b)
    assert err == 0
    ch = np.nonzero(idx != base)[0] // 3
    assert ch.size and np.all((ch >= r["tri_base"]) & (ch < r["tri_base"] + r["Tp"]))
    # GTS index out of range -> INDEX error
    e1 = orc.encode(m, 32, 48, 1)
    r1 = read_records(e1.blob)[2]
    b = e1.blob.copy()
    W = (r1["Tp"] + 31) // 32
    b[r1["offset"] + r1["hdr"] + 4 * W] = 255
    err, errs, *_ = orc.decode(b)
    assert errs[2] & orc.DERR_INDEX
    # record size mismatch -> RECORD error
    bad = pack_meshlets(orc, 1, [gts_meshlet(4, [1], [3] * 20)])
    err, errs, *_ = orc.decode(bad)
    assert errs[0] & orc.DERR_RECORD


def test_encoder_rejects_degenerate_source(orc):
    m = synth.quad_grid(2, 2)
    idx = m.indices.copy()
    idx[0, 1] = idx[0, 0]
    with pytest.raises(ValueError):
        orc.encode(synth.Mesh(idx, m.attributes, m.bits, m.semantic), 64, 126, 2)


def test_checksum_additivity(orc):
    rng = np.random.default_rng(0)
    w = rng.integers(0, 2**32, size=1000, dtype=np.uint64).astype(np.uint32)
    full = orc.checksum(w, 0)
    parts = (orc.checksum(w[:313], 0) + orc.checksum(w[313:], 313)) % 2**64
    assert full == parts


def test_checksum_splitmix64_vectors(orc):
    """FORMAT.md §6's mix64 is the SplitMix64 finaliser; the published
    SplitMix64 sequence for seed 0 is mix64(i * 0x9e3779b97f4a7c15) for i = 1, 2, 3:
    0xe220a8397b1dcdaf, 0x6e789e6aa1b965f4, 0x06c45d188009454f.  A one-word buffer at word
    index k holding w contributes mix64(k << 32 | w), so choosing (k, w) as the halves of
    i * golden must reproduce those published values."""
    golden = 0x9E3779B97F4A7C15
    want = [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    for i, v in enumerate(want, start=1):
        z = (golden * i) % 2**64
        k, w = z >> 32, z & 0xFFFFFFFF
        assert orc.checksum(np.array([w], np.uint32), k) == v
