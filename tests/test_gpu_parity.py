"""GPU parity: the sm_100a decoder (through the C ABI) against the oracle's sequential decode.

Bar (BASELINE north_star): indices and quantised attributes bit-exact; fp32 attributes
0 ULP (compared as bit patterns); checksums equal the oracle's.  Inputs are seeded and
synthetic; expected values come only from oracle/ (never from the CUDA path).
"""
import itertools

import numpy as np
import pytest

import synth
from streams import gts_meshlet, pack_meshlets, read_records, reuse_meshlet

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


def gpu_vs_oracle(mc, orc, blob_bytes, want_q=True, flags=0, check_stats=True):
    blob_bytes = np.ascontiguousarray(blob_bytes)
    db = mc.DeviceBlob(blob_bytes, want_vertices=True, want_quantized=want_q)
    st = db.decode_stats(flags=flags)
    torch.cuda.synchronize()
    err, errs, idx, q, f = orc.decode(blob_bytes, want_q=want_q)
    L = db.layout
    if flags & mc.MC_DECODE_BLOB_LOCAL_INDICES:
        idx = (idx.astype(np.int64) - L.base_vtx).astype(np.uint32)
    assert err == 0 and st["error_bits"] == 0, (err, st)
    np.testing.assert_array_equal(_u32(db.indices), idx)
    if want_q:
        np.testing.assert_array_equal(_u32(db.quantized), q)
    np.testing.assert_array_equal(_u32(db.vertices), f.view(np.uint32))
    if check_stats:
        assert st["checksum_indices"] == orc.checksum(idx, 3 * L.base_tri)
        assert st["checksum_vertices"] == orc.checksum(f, L.n_out * L.base_vtx)
        if want_q:
            assert st["checksum_quantized"] == orc.checksum(q, L.n * L.base_vtx)
        assert st["triangles"] == L.total_tp and st["vertices"] == L.total_v
        tri = idx.reshape(-1, 3)
        deg = (tri[:, 0] == tri[:, 1]) | (tri[:, 1] == tri[:, 2]) | (tri[:, 0] == tri[:, 2])
        assert st["degenerate"] == int(deg.sum())
    # the timed (non-stats) kernel writes the same bytes
    db2 = mc.DeviceBlob(blob_bytes, want_vertices=True, want_quantized=want_q)
    db2.decode(flags=flags)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(_u32(db2.indices), _u32(db.indices))
    np.testing.assert_array_equal(_u32(db2.vertices), _u32(db.vertices))
    return db, st


# ------------------------------------------------------------------ oracle-encoded scenes

@pytest.mark.parametrize("codec", [1, 2])
@pytest.mark.parametrize("limits", [(64, 126), (128, 256), (32, 32), (256, 256), (3, 1)])
def test_cfg1_grid_oracle_encoded(mc, orc, codec, limits):
    e = orc.encode(synth.quad_grid(32, 32), *limits, codec)
    gpu_vs_oracle(mc, orc, e.blob)


@pytest.mark.parametrize("seed", range(6))
def test_random_patches_generic_layout(mc, orc, seed):
    """n=5 generic channels with random widths 3..24 bits: the runtime-layout kernel."""
    m = synth.random_patch(seed, nx=30, ny=20)
    for codec in (1, 2):
        gpu_vs_oracle(mc, orc, orc.encode(m, [64, 32, 128][seed % 3], [126, 64, 256][seed % 3], codec).blob)


@pytest.mark.parametrize("bits", [8, 10, 12, 16, 20, 24])
def test_bit_widths_cfg5(mc, orc, bits):
    m = synth.displaced_sphere(20, bits=bits)
    gpu_vs_oracle(mc, orc, orc.encode(m, 64, 126, 2).blob)
    m8 = synth.quad_grid(24, 24, bits=bits)
    gpu_vs_oracle(mc, orc, orc.encode(m8, 128, 256, 1).blob)


def test_layouts(mc, orc):
    """Every kernel instantiation: n=8 (pos3+nrm3+uv2), n=7 oct, n=3, generic oct placement."""
    gpu_vs_oracle(mc, orc, orc.encode(synth.torus(60, 30), 64, 126, 2).blob)
    gpu_vs_oracle(mc, orc, orc.encode(synth.displaced_sphere(15), 64, 126, 2).blob)
    gpu_vs_oracle(mc, orc, orc.encode(synth.displaced_sphere(15, oct_normals=False), 64, 126, 1).blob)
    m = synth.displaced_sphere(12)
    attr = np.concatenate([m.attributes[:, 5:7], m.attributes[:, 3:5], m.attributes[:, 0:3]], 1)
    m2 = synth.Mesh(m.indices, attr, [12, 13, 16, 16, 9, 10, 11], [3, 3, 4, 4, 1, 1, 1])
    gpu_vs_oracle(mc, orc, orc.encode(m2, 64, 126, 2).blob)


# ------------------------------------------------------------------ exhaustive tiny streams

def test_exhaustive_tiny_gts(mc, orc):
    """Every GTS stream with T' <= 6 and V <= 6 (all flags x all indices, SURVEY §8(c)
    "tiny meshlets"), one launch: 429,344 records."""
    ms = []
    for Tp in range(1, 7):
        for V in range(3, 7):
            for flags in itertools.product([0, 1], repeat=Tp - 1):
                for idx in itertools.product(range(V), repeat=Tp - 1):
                    ms.append(gts_meshlet(V, flags, idx))
    assert len(ms) == sum(2 ** (Tp - 1) * V ** (Tp - 1) for Tp in range(1, 7) for V in range(3, 7))
    assert len(ms) > 400000
    rng = np.random.default_rng(0)
    codes = rng.integers(0, 256, size=sum(m["V"] for m in ms))
    blob = pack_meshlets(orc, 1, ms, codes=codes, vmax=6, tmax=6)
    gpu_vs_oracle(mc, orc, blob)


def test_exhaustive_tiny_reuse(mc, orc):
    """Every GTS-Reuse stream with T' <= 6, V <= 6: all increment patterns with
    popcount V-3, all reuse values, all L/R flags."""
    ms = []
    for Tp in range(1, 7):
        for inc in itertools.product([0, 1], repeat=Tp - 1):
            V = 3 + sum(inc)
            if V > 6:
                continue
            nz = (Tp - 1) - sum(inc)
            for flags in itertools.product([0, 1], repeat=Tp - 1):
                for reuse in itertools.product(range(V), repeat=nz):
                    ms.append(reuse_meshlet(V, flags, inc, reuse))
    assert len(ms) > 20000
    blob = pack_meshlets(orc, 2, ms, vmax=6, tmax=6)
    gpu_vs_oracle(mc, orc, blob)


def test_long_fans_multiword(mc, orc):
    """Random T' up to 256 with long same-flag runs crossing words, both codecs."""
    rng = np.random.default_rng(7)
    ms = []
    for k in range(400):
        Tp = int(rng.integers(1, 257))
        f, cur = [], int(rng.integers(0, 2))
        while len(f) < Tp - 1:
            run = int(rng.integers(1, 120))
            f += [cur] * run
            cur ^= 1
        ms.append(gts_meshlet(256, f[:Tp - 1], rng.integers(0, 256, size=Tp - 1)))
    db, st = gpu_vs_oracle(mc, orc, pack_meshlets(orc, 1, ms, vmax=256, tmax=256))
    assert st["multiword_lookbacks"] > 0 and st["max_lookback"] > 64
    m = synth.fan(254, n_ch=3)
    gpu_vs_oracle(mc, orc, orc.encode(m, 256, 256, 2).blob)


def test_max_sizes(mc, orc):
    """Ṽ = T̃ = 256, n = 16 channels at 24 bits (largest record), generic kernel."""
    rng = np.random.default_rng(3)
    M = 300
    ms, codes = [], []
    for k in range(M):
        Tp = 256 if k % 2 == 0 else int(rng.integers(1, 257))
        V = 256 if k % 3 else int(rng.integers(3, 257))
        ms.append(gts_meshlet(V, rng.integers(0, 2, size=Tp - 1), rng.integers(0, V, size=Tp - 1)))
        codes.append(rng.integers(0, 2**24, size=V * 16))
    bits = [24] * 16
    L = rng.integers(0, 2**31, size=M * 16)
    delta = rng.uniform(1e-6, 1e-3, size=16).astype(np.float32)
    origin = rng.uniform(-100, 100, size=16).astype(np.float32)
    blob = pack_meshlets(orc, 1, ms, n=16, bits=bits, codes=np.concatenate(codes), L=L, delta=delta,
                         origin=origin, vmax=256, tmax=256)
    gpu_vs_oracle(mc, orc, blob)


@pytest.mark.parametrize("n,sem", [(7, [1, 1, 1, 4, 4, 3, 3]), (8, [1, 1, 1, 2, 2, 2, 3, 3]), (3, [1, 1, 1])])
@pytest.mark.parametrize("b", [16, 12])
def test_int_to_float_boundary(mc, orc, n, sem, b):
    """Grid values q = L_c + code on both sides of 2^23: records whose every q < 2^23 take the
    exact bit-trick conversion (0x4B000000 + q as a float, minus 2^23), the others the
    conversion instruction; both must give the oracle's (float)q bit for bit (FORMAT.md §4)."""
    rng = np.random.default_rng(11 + n + b)
    bm = (1 << b) - 1
    M = 240
    ms, codes, L = [], [], []
    edge = (1 << 23) - 1 - bm
    for k in range(M):
        Tp = int(rng.integers(1, 127))
        V = int(rng.integers(3, 65))
        ms.append(gts_meshlet(V, rng.integers(0, 2, size=Tp - 1), rng.integers(0, V, size=Tp - 1)))
        c = rng.integers(0, bm + 1, size=V * n)
        if k % 4 == 0:
            c[rng.integers(0, V * n)] = bm                        # largest code present
        codes.append(c)
        mode = k % 6
        if mode == 0:
            Lk = np.full(n, edge)                                 # q reaches 2^23 - 1: fast path
        elif mode == 1:
            Lk = np.full(n, edge); Lk[rng.integers(0, n)] += 1    # one channel may reach 2^23
        elif mode == 2:
            Lk = rng.integers(0, edge + 1, size=n)
        elif mode == 3:
            Lk = rng.integers(edge - 5, edge + 6, size=n)
        elif mode == 4:
            Lk = rng.integers(1 << 23, 1 << 28, size=n)           # large q: conversion instruction
        else:
            Lk = rng.integers(0, 1 << 12, size=n)
        L.append(Lk)
    delta = np.full(n, 1e-7, np.float32)
    origin = np.full(n, -0.5, np.float32)
    blob = pack_meshlets(orc, 1, ms, n=n, bits=[b] * n, sem=sem, codes=np.concatenate(codes),
                         L=np.concatenate(L).astype(np.uint32), delta=delta, origin=origin, vmax=64, tmax=126)
    gpu_vs_oracle(mc, orc, blob)


def test_empty_and_ragged(mc, orc):
    e = orc.encode(synth.quad_grid(2, 1), 64, 126, 2)
    gpu_vs_oracle(mc, orc, e.blob)
    empty = pack_meshlets(orc, 2, [], vmax=64, tmax=126)
    db = mc.DeviceBlob(empty)
    st = db.decode_stats()
    assert st["triangles"] == 0 and st["error_bits"] == 0
    # sub-ranges: only the range's outputs are written
    e = orc.encode(synth.torus(40, 20), 64, 126, 2)
    db = mc.DeviceBlob(e.blob, want_quantized=True)
    db.indices.fill_(-1)
    db.decode(first=3, count=5)
    torch.cuda.synchronize()
    err, errs, idx, q, f = orc.decode(e.blob)
    recs = read_records(e.blob)
    lo, hi = recs[3]["tri_base"], recs[8]["tri_base"]
    got = _u32(db.indices)
    np.testing.assert_array_equal(got[3 * lo:3 * hi], idx[3 * lo:3 * hi])
    assert np.all(got[:3 * lo] == 0xFFFFFFFF) and np.all(got[3 * hi:] == 0xFFFFFFFF)


# ------------------------------------------------------------------ product encoder + sharding + e2e

@pytest.mark.parametrize("codec", [1, 2])
def test_product_encoded_scenes(mc, orc, codec):
    for m, lim in [(synth.quad_grid(), (64, 126)), (synth.torus(300, 150), (64, 126)),
                   (synth.displaced_sphere(60), (128, 256)), (synth.random_patch(11, 40, 30), (32, 32))]:
        b = mc.mc_encode(m, *lim, codec)
        gpu_vs_oracle(mc, orc, np.array(b.bytes))


def test_shards_sum_to_whole(mc, orc):
    b = mc.mc_encode(synth.displaced_sphere(50), 64, 126, 2)
    full = np.array(b.bytes)
    dbf, stf = gpu_vs_oracle(mc, orc, full)
    tot_i = tot_f = 0
    cat = []
    for f0, c in b.shard_ranges(8):
        s = b.extract(f0, c)
        db, st = gpu_vs_oracle(mc, orc, np.array(s.bytes))
        tot_i = (tot_i + st["checksum_indices"]) % 2**64
        tot_f = (tot_f + st["checksum_vertices"]) % 2**64
        cat.append(_u32(db.indices))
        db2, _ = gpu_vs_oracle(mc, orc, np.array(s.bytes), flags=mc.MC_DECODE_BLOB_LOCAL_INDICES,
                               check_stats=False)
    assert tot_i == stf["checksum_indices"] and tot_f == stf["checksum_vertices"]
    np.testing.assert_array_equal(np.concatenate(cat), _u32(dbf.indices))


@pytest.mark.parametrize("chunks", [0, 2, 7, 64])
@pytest.mark.parametrize("index_format", ["u32", "u8x4"])
def test_decode_host_e2e(mc, orc, chunks, index_format):
    """mc_decode_host from pinned host buffers, serial (chunks 0) and pipelined over PCIe
    (chunks >= 2, more chunks than some records): bit-exact with the oracle; the outputs
    are poisoned first so a chunk whose copy-out is missing or misplaced shows up."""
    b = mc.mc_encode(synth.torus(100, 50), 64, 126, 2)
    data = np.array(b.bytes)
    L = mc.parse_header(data)
    u8 = index_format == "u8x4"
    flags = mc.MC_DECODE_INDEX_LOCAL_U8X4 if u8 else 0
    nidx = (1 if u8 else 3) * L.total_tp
    h_blob = torch.from_numpy(data).pin_memory()
    h_idx = torch.full((nidx,), -1, dtype=torch.int32).pin_memory()
    h_v = torch.full((L.n_out * L.total_v,), -1, dtype=torch.int32).pin_memory().view(torch.float32)
    h_q = torch.full((L.n * L.total_v,), -1, dtype=torch.int32).pin_memory()
    d_blob = torch.zeros(data.nbytes, dtype=torch.uint8, device="cuda")
    d_idx = torch.empty(nidx, dtype=torch.int32, device="cuda")
    d_v = torch.empty(L.n_out * L.total_v, dtype=torch.float32, device="cuda")
    d_q = torch.empty(L.n * L.total_v, dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    mc.mc_decode_host(L, h_blob, d_blob, h_idx, d_idx, h_v, d_v, h_q, d_q, flags=flags, stream=s, chunks=chunks)
    s.synchronize()                      # ordered on the caller's stream, copy streams included
    err, errs, idx, q, f = orc.decode(data)
    assert err == 0
    if u8:
        err8, idx = orc.decode_u8x4(data)
        assert err8 == 0
    np.testing.assert_array_equal(h_idx.numpy().view(np.uint32), idx)
    np.testing.assert_array_equal(h_v.numpy().view(np.uint32), f.view(np.uint32))
    np.testing.assert_array_equal(h_q.numpy().view(np.uint32), q)


# ------------------------------------------------------------------ malformed streams (FORMAT.md §5)

def test_malformed_streams_flagged(mc, orc):
    m = synth.quad_grid(16, 16)
    for codec, what in ((2, "inc"), (1, "idx"), (2, "reuse"), (1, "size"), (2, "object")):
        e = orc.encode(m, 32, 48, codec)
        b = e.blob.copy()
        recs = read_records(b)
        k = 5
        r = recs[k]
        W = (r["Tp"] + 31) // 32
        if what == "inc":
            b[r["offset"] + r["hdr"] + 4 * W] ^= 0x02
        elif what == "idx":
            b[r["offset"] + r["hdr"] + 4 * W] = 250
        elif what == "reuse":
            nb = (r["Tp"] - 1) - (r["V"] - 3)
            assert nb > 0
            b[r["offset"] + r["hdr"] + 8 * W] = 250
        elif what == "size":
            b[r["offset"] + 8] = (r["V"] - 1) + 5           # 5 more vertices: +80 B of attributes
        elif what == "object":
            b[r["offset"] + 10] = 7
        err, errs, *_ = orc.decode(b)
        assert err != 0
        db = mc.DeviceBlob(b)
        st = db.decode_stats()
        assert st["error_bits"] == err, (what, st["error_bits"], err)
        assert st["first_bad_meshlet"] == int(np.nonzero(errs)[0][0])
        assert st["num_bad"] == int(np.count_nonzero(errs))
