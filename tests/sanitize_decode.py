"""Decode workloads through the product path for compute-sanitizer (tests/test_gpu_sanitizer.py).
Test infrastructure: the exhaustive tiny streams are serialised with the oracle's packer.

    compute-sanitizer --tool memcheck|racecheck|synccheck python tests/sanitize_decode.py [--big]

Covers: the cfg1 grid (GTS, GTS-Reuse, Basic; stats and timed kernels; u32 and u8x4), every
GTS-Reuse stream with T' <= 5 and V <= 6, long multi-word fans at T~ = 256 (32-lane groups),
a generic-layout blob (bit reader), a cone-culled compacted decode (cull reduce / scan /
emit + list decode), the static-stride short-launch kernel, and with --big one
dynamic-claim launch (>= 60k records).  Exits non-zero on any decode error bit."""
import itertools
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

import paper_2404_06359_b200 as mc  # noqa: E402
import synth  # noqa: E402


def run(blob, fmt="u32", stats=True, culled=False):
    db = mc.DeviceBlob(blob, want_vertices=True, want_quantized=True, index_format=fmt)
    db.decode()
    bad = 0
    if stats:
        bad |= db.decode_stats()["error_bits"]
    if culled:
        d = np.array([1.0, 2.0, -3.0]) / np.sqrt(14.0)
        bad |= db.decode_culled(d.astype(np.float32), stats=True)["error_bits"]
    torch.cuda.synchronize()
    return bad


def main():
    big = "--big" in sys.argv
    torch.cuda.set_device(0)
    bad = 0
    grid = synth.quad_grid(32, 32)
    for codec in (1, 2, 3):
        b = mc.mc_encode(grid, 64, 126, codec)
        bad |= run(b) | run(b, "u8x4")
    # every GTS-Reuse stream with T' <= 5, V <= 6 (oracle packer: raw streams)
    import oracle
    from streams import pack_meshlets, reuse_meshlet
    ms = []
    for Tp in range(1, 6):
        for inc in itertools.product([0, 1], repeat=Tp - 1):
            V = 3 + sum(inc)
            if V > 6:
                continue
            for flags in itertools.product([0, 1], repeat=Tp - 1):
                for reuse in itertools.product(range(V), repeat=(Tp - 1) - sum(inc)):
                    ms.append(reuse_meshlet(V, flags, inc, reuse))
    bad |= run(pack_meshlets(oracle, 2, ms, vmax=6, tmax=6))
    # long fans crossing flag words, T~ = 256 (32-lane groups), generic layout
    bad |= run(mc.mc_encode(synth.fan(254, n_ch=3), 256, 256, 2))
    bad |= run(mc.mc_encode(synth.random_patch(2, nx=40, ny=30), 128, 256, 1))
    bad |= run(mc.mc_encode(synth.quad_grid(24, 24, bits=12), 32, 32, 2))
    # culled decode (cones from the product encoder)
    bad |= run(mc.mc_encode(synth.displaced_sphere(30), 64, 126, 2, cull_cones=True), culled=True)
    # static-stride kernel (u32, compile-time layout, short launch)
    bad |= run(mc.mc_encode(synth.torus(200, 100), 64, 126, 2), stats=False)
    if big:   # one dynamic-claim launch
        protos = [mc.mc_encode(synth.building(12, s), 64, 126, 2) for s in range(3)]
        n = 60000 // protos[0].layout.num_meshlets + 1
        rng = np.random.default_rng(0)
        blob = mc.mc_blob_instance(protos, rng.integers(0, 3, n).astype(np.uint32),
                                   rng.uniform(-9, 9, (n, 3)).astype(np.float32))
        bad |= run(blob, stats=False) | run(blob, "u8x4", stats=False)
    if "--fuzz" in sys.argv:
        fuzz()
    print("decode error bits:", bad)
    sys.exit(1 if bad else 0)


def fuzz(rounds: int = 40):
    """Random byte corruption inside the records section (header and directory intact, so
    the blob parses): every kernel must stay inside its buffers whatever the records hold
    (error bits are expected and not counted)."""
    rng = np.random.default_rng(7)
    blobs = [mc.mc_encode(synth.quad_grid(32, 32), 64, 126, c) for c in (1, 2, 3)]
    blobs += [mc.mc_encode(synth.quad_grid(24, 24, bits=12), 32, 32, 2),
              mc.mc_encode(synth.random_patch(3, nx=30, ny=20), 128, 256, 2),
              mc.mc_encode(synth.quad_grid(32, 32), 64, 126, 2, variable_widths=True)]
    for r in range(rounds):
        src = blobs[r % len(blobs)]
        data = np.array(src.bytes).copy()
        L = src.layout
        lo = int(L.off_rec)
        k = int(rng.integers(1, 64))
        pos = rng.integers(lo, data.size, k)
        data[pos] ^= rng.integers(1, 256, k).astype(np.uint8)
        blob = mc.Blob.from_bytes(data)
        for fmt in ("u32", "u8x4"):
            db = mc.DeviceBlob(blob, want_vertices=True, want_quantized=True, index_format=fmt)
            db.decode()
            db.decode_stats()
    torch.cuda.synchronize()
    print("fuzz rounds:", rounds)


if __name__ == "__main__":
    main()
