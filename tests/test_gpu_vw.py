"""GPU parity for per-meshlet attribute widths (FORMAT.md VW).

Indices bit-exact, q bit-exact, fp32 0 ULP and checksums equal to the oracle's
sequential decode, for the compiled layouts (pos3+nrm3+uv2, pos3+oct2+uv2, pos3) and
the generic kernel, every codec, both index formats, stats and timed kernels.
"""
import numpy as np
import pytest

import synth
from streams import read_records
from test_gpu_basic_u8x4 import check

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2404_06359_b200 as mc
    mc.lib()
    return mc


MESHES = {
    "nrm8ch": lambda: synth.displaced_sphere(40, oct_normals=False),         # layout 1
    "oct7ch": lambda: synth.displaced_sphere(40),                            # layout 2
    "pos3": lambda: synth.torus(120, 60),                                    # layout 3
    "generic": lambda: synth.random_patch(3, 30, 20),                        # mixed widths
    "bits10": lambda: synth.displaced_sphere(30).with_bits(10),
}


@pytest.mark.parametrize("name", list(MESHES))
@pytest.mark.parametrize("codec", [1, 2, 3])
def test_vw_parity(mc, orc, name, codec):
    m = MESHES[name]()
    for lim in ((64, 126), (256, 256)):
        b = np.array(mc.mc_encode(m, *lim, codec, variable_widths=True).bytes)
        check(mc, orc, b)


@pytest.mark.parametrize("codec", [2, 3])
def test_vw_u8x4_and_oracle_encoded(mc, orc, codec):
    m = MESHES["oct7ch"]()
    check(mc, orc, np.array(mc.mc_encode(m, 64, 126, codec, variable_widths=True).bytes), index_format="u8x4",
          want_q=False)
    check(mc, orc, orc.encode(m, 64, 126, codec, vw=True).blob)


def test_vw_city_instances(mc, orc):
    scene = synth.city(num_instances=5, num_prototypes=2, k=14)
    protos = [mc.mc_encode(p, 64, 126, 2, variable_widths=True) for p in scene.prototypes]
    blob = mc.mc_blob_instance_range(protos, scene.instance_proto, scene.instance_offset, 1, 3)
    check(mc, orc, np.array(blob.bytes))


def test_vw_width_fault(mc, orc):
    """A record width above b_c is a RECORD error on both sides (FORMAT.md §5)."""
    e = orc.encode(MESHES["oct7ch"](), 64, 126, 2, vw=True)
    blob = e.blob.copy()
    r = read_records(blob)[2]
    n = orc.blob_info(blob).n
    blob[r["offset"] + 16 + 4 * n + 1] = 17
    err, errs, idx, q, f = orc.decode(blob)
    db = mc.DeviceBlob(blob)
    st = db.decode_stats()
    assert err == orc.DERR_RECORD and st["error_bits"] == orc.DERR_RECORD and st["first_bad_meshlet"] == 2
