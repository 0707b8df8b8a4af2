"""GPU parity of every timed kernel instantiation AT THE LAUNCH SIZE WHERE IT DISPATCHES.

decode.cu picks a kernel per launch: the static-stride short-launch kernel (u32 output,
compile-time halfword layout, fewer than MC_STATIC_BELOW records per group of a full
grid: < 56,832 records on 148 SMs), the dynamic-claim kernels above that (the u8x4-only
build for the strip codecs' u8x4 output), 8-lane groups with K = 1 flag word for T~ <= 32,
16-lane groups with K = 2 for T~ <= 64 and K = 4 for T~ <= 128, 32-lane groups for
T~ > 128, the bit reader (widths != 16) and the
per-meshlet-width reader (VW).  Each case below builds a blob of the size that selects the
kernel (instanced small prototypes: >= 60,000 records for the dynamic kernels) and compares
the NON-stats decode (the timed path) element by element with the oracle's sequential
decode: u32 indices, u8x4 words, fp32 vertex bit patterns.
"""
import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ST_LIMIT = 8 * 148 * 3 * 16      # MC_STATIC_BELOW x SMs x CTAs/SM x 16 groups per CTA


@pytest.fixture(scope="module")
def mc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2404_06359_b200 as mc
    mc.lib()
    return mc


def _protos(layout: str, bits: int = 16):
    if layout == "n7oct":        # pos3 + oct2 + uv2 (cfg3/cfg4)
        return [synth.building(12, s, bits) for s in range(3)]
    if layout == "n8":           # pos3 + nrm3 + uv2 (the paper's 8 attributes)
        return [synth.displaced_sphere(12, seed=s, oct_normals=False, bits=bits) for s in range(3)]
    if layout == "n3":           # positions only (cfg2)
        return [synth.torus(48 + 8 * s, 24, bits=bits) for s in range(3)]
    raise ValueError(layout)


def _instanced(mc, layout, codec, limits, min_records, bits=16, vw=False):
    protos = [mc.mc_encode(p, *limits, codec, variable_widths=vw) for p in _protos(layout, bits)]
    per = sum(p.layout.num_meshlets for p in protos) / len(protos)
    n_inst = int(np.ceil(min_records / per))
    rng = np.random.default_rng(1)
    proto_of = rng.integers(0, len(protos), n_inst).astype(np.uint32)
    off = rng.uniform(-50, 50, size=(n_inst, 3)).astype(np.float32)
    blob = mc.mc_blob_instance(protos, proto_of, off)
    assert blob.layout.num_meshlets >= min_records
    return blob


def _check(mc, orc, blob, index_format):
    data = np.array(blob.bytes)
    db = mc.DeviceBlob(blob, want_vertices=True, want_quantized=False, index_format=index_format)
    db.indices.fill_(-1)
    db.vertices.fill_(float("nan"))
    db.decode()                                   # the timed (non-stats) kernel
    torch.cuda.synchronize()
    gi = db.indices.cpu().numpy().view(np.uint32)
    gf = db.vertices.cpu().numpy().view(np.uint32)
    err, errs, idx, q, f = orc.decode(data, want_q=False)
    assert err == 0
    if index_format == "u8x4":
        e2, words = orc.decode_u8x4(data)
        assert e2 == 0
        np.testing.assert_array_equal(gi, words)
    else:
        np.testing.assert_array_equal(gi, idx)
    np.testing.assert_array_equal(gf, f.view(np.uint32))


@pytest.mark.parametrize("fmt", ["u32", "u8x4"])
@pytest.mark.parametrize("layout", ["n3", "n7oct", "n8"])
@pytest.mark.parametrize("codec", [1, 2, 3])
def test_dynamic_kernels_64_126(mc, orc, codec, layout, fmt):
    """>= 60k records at 64v/126t: the dynamic-claim kernel (u8x4-only build for GTS /
    GTS-Reuse u8x4, the run-time-format kernel otherwise)."""
    _check(mc, orc, _instanced(mc, layout, codec, (64, 126), 60000), fmt)


@pytest.mark.parametrize("layout", ["n3", "n7oct", "n8"])
@pytest.mark.parametrize("codec", [1, 2, 3])
def test_static_stride_kernel(mc, orc, codec, layout):
    """< 56,832 records, u32 output: the static-stride short-launch kernel."""
    blob = _instanced(mc, layout, codec, (64, 126), 20000)
    assert blob.layout.num_meshlets < ST_LIMIT
    _check(mc, orc, blob, "u32")


@pytest.mark.parametrize("fmt", ["u32", "u8x4"])
@pytest.mark.parametrize("limits", [(32, 32), (64, 64), (128, 256), (256, 256)])
@pytest.mark.parametrize("codec", [1, 2])
def test_group_shapes(mc, orc, codec, limits, fmt):
    """T~ <= 32 (8-lane groups, one flag word per step), T~ <= 64 (16-lane groups, two flag
    words per step) and T~ > 128 (32-lane groups)."""
    _check(mc, orc, _instanced(mc, "n7oct", codec, limits, 60000), fmt)


@pytest.mark.parametrize("layout,bits", [("n3", 8), ("n3", 12), ("n3", 24), ("n8", 8), ("n8", 10), ("n8", 12),
                                         ("n8", 20), ("n8", 24)])
@pytest.mark.parametrize("limits", [(64, 126), (32, 32), (128, 256)])
def test_bit_reader_kernels(mc, orc, layout, bits, limits):
    """Widths != 16 at the dynamic launch size: n = 8 with one width for every channel takes
    the compile-time unpack (units of word-aligned vertices), n = 3 the run-time funnel-shift
    bit reader."""
    _check(mc, orc, _instanced(mc, layout, 2, limits, 60000, bits=bits), "u32")


@pytest.mark.parametrize("codec", [1, 3])
def test_uniform_width_other_codecs(mc, orc, codec):
    _check(mc, orc, _instanced(mc, "n8", codec, (64, 126), 60000, bits=10), "u8x4")


@pytest.mark.parametrize("fmt", ["u32", "u8x4"])
@pytest.mark.parametrize("codec", [1, 2])
def test_vw_kernels(mc, orc, codec, fmt):
    """Per-meshlet widths (FORMAT.md VW) at the dynamic launch size."""
    _check(mc, orc, _instanced(mc, "n7oct", codec, (64, 126), 60000, vw=True), fmt)


@pytest.mark.parametrize("layout", ["n7oct", "n8"])
def test_vertices_16b_aligned_output(mc, orc, layout):
    """n_out = 8 vertices leave with one 256-bit store when d_vertices is 32-B aligned; a
    buffer that is only 16-B aligned (the ABI's minimum) takes the two 128-bit stores.
    Both at a dynamic-kernel launch size, element by element against the oracle."""
    blob = _instanced(mc, layout, 2, (64, 126), 60_000)
    data = np.array(blob.bytes)
    L = blob.layout
    d_blob = torch.from_numpy(data).cuda()
    idx = torch.empty(3 * L.total_tp, dtype=torch.int32, device="cuda")
    raw = torch.full((8 * L.total_v + 4,), float("nan"), dtype=torch.float32, device="cuda")
    assert raw.data_ptr() % 32 == 0
    err, errs, ridx, q, f = orc.decode(data, want_q=False)
    assert err == 0
    for off in (4, 0):                            # +16 B: not 32-B aligned; 0: aligned
        verts = raw[off:off + 8 * L.total_v]
        verts.fill_(float("nan"))
        mc.mc_decode_meshlets(L, d_blob, idx, verts)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(idx.cpu().numpy().view(np.uint32), ridx)
        np.testing.assert_array_equal(verts.cpu().numpy().view(np.uint32), f.view(np.uint32))
