"""CPU checks of bench.py's host logic: shard splits, algorithmic bytes,
the shared config dict of both arms, the ncu-traffic key per launch shape."""
import argparse
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_split_range_tiles_and_balances():
    import bench
    for total in (1, 7, 125, 1000, 1001):
        for world in (1, 2, 3, 8):
            parts = [bench.split_range(total, r, world) for r in range(world)]
            assert parts[0][0] == 0
            for (f0, c0), (f1, _) in zip(parts, parts[1:]):
                assert f0 + c0 == f1
            assert sum(c for _, c in parts) == total
            assert max(c for _, c in parts) - min(c for _, c in parts) <= 1


def test_algorithmic_bytes_from_records():
    """Record bytes read + directory + object table + 12 (or 4) B per decoded triangle +
    4 n_out B per vertex, restated from the records read by tests/streams.py."""
    import bench
    import paper_2404_06359_b200 as mc
    import synth
    from streams import read_records
    blob = mc.mc_encode(synth.displaced_sphere(12), 64, 126, 2)
    L = blob.layout
    recs = read_records(np.array(blob.bytes))
    rec_bytes = sum(r["size"] for r in recs)
    want = rec_bytes + 4 * (len(recs) + 1) + 8 * L.n * L.num_objects + \
        sum(12 * r["Tp"] + 4 * L.n_out * r["V"] for r in recs)
    assert bench.algorithmic_bytes(L, "u32") == want
    want8 = want - sum(8 * r["Tp"] for r in recs)
    assert bench.algorithmic_bytes(L, "u8x4") == want8


def _args(**kw):
    d = dict(workload="cfg4_city", codec=2, index_format="u32", variable_widths=False, cull=False,
             instances=1000, scaling="strong")
    d.update(kw)
    return argparse.Namespace(**d)


def test_config_dict_identical_for_both_arms():
    import bench
    import paper_2404_06359_b200 as mc
    blob, meta = bench.build_blob(mc, "cfg4_city", 0, 1, 2, 3, protos_k=(2, 8))
    L = blob.layout
    alg = bench.algorithmic_bytes(L, "u32")
    a = bench.config_dict(_args(instances=3), L, meta, 1, alg, alg < 4 * bench.L2_BYTES)
    b = bench.config_dict(_args(instances=3), L, meta, 1, alg, alg < 4 * bench.L2_BYTES)
    assert a == b and a["workload"] == "cfg4_city" and a["scaling"] == "strong"
    assert "model" not in a


def test_ncu_traffic_key_per_launch_shape():
    import bench
    t, src = bench.ncu_traffic(_args(), 1)
    t8, src8 = bench.ncu_traffic(_args(), 8)
    t125, src125 = bench.ncu_traffic(_args(instances=125), 1)
    assert src is not None and src8 is not None and src8 == src125 and t8 == t125 and t8 < t
    assert bench.ncu_traffic(_args(instances=77), 1) == (None, None)
