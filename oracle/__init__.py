"""Test oracle for per-meshlet decompression — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline``
leg and ``--impl reference``) may import this package.  The product package
``paper_2404_06359_b200`` never imports it and shares no code with it; both sides
implement ``FORMAT.md`` independently.

The arithmetic lives in plain C (``oracle/oracle.c``, compiled with
``-ffp-contract=off``); this module only marshals numpy arrays through ctypes.
See ``oracle/oracle.c`` for the paper passages each function follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

DERR_RECORD, DERR_COUNTS, DERR_INDEX, DERR_REUSE, DERR_OBJECT = 1, 2, 4, 8, 16
CODEC_GTS, CODEC_REUSE, CODEC_BASIC = 1, 2, 3


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc (no intrinsics, no contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math",
                               "-fPIC", "-shared", "-Wall", "-Wno-unused-function",
                               "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        u32, u64, sz = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_size_t
        L.or_blob_info.argtypes = [P, sz, P]
        L.or_decode_meshlet.argtypes = [P, sz, u32, P, P, P, P]
        L.or_decode_meshlet.restype = u32
        L.or_decode_range.argtypes = [P, sz, u32, u32, P, P, P, P]
        L.or_decode_range.restype = u32
        L.or_decode_range_u8x4.argtypes = [P, sz, u32, u32, P]
        L.or_decode_range_u8x4.restype = u32
        L.or_decode_culled.argtypes = [P, sz, P, u32, P, P, P, P, P]
        L.or_decode_culled.restype = u32
        L.or_add_cull.argtypes = [P, sz, P, ctypes.POINTER(P), ctypes.POINTER(u64)]
        L.or_checksum.argtypes = [P, u64, u64]
        L.or_checksum.restype = u64
        L.or_oct_decode.argtypes = [ctypes.c_float, ctypes.c_float, P]
        L.or_encode.argtypes = [P, u32, P, u32, u32, P, P, P, u32, u32, u32, u32,
                                ctypes.POINTER(P), ctypes.POINTER(u64), ctypes.POINTER(P),
                                ctypes.POINTER(P), P]
        L.or_pack.argtypes = [u32, u32, P, P, u32, P, P, u32, u32, u32, P, P, P, P, P, P, P, P, P, P,
                              ctypes.POINTER(P), ctypes.POINTER(u64)]
        L.or_free.argtypes = [P]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


class Info(dict):
    __getattr__ = dict.__getitem__


def blob_info(blob: np.ndarray) -> Info:
    out = np.zeros(16, np.uint32)
    st = lib().or_blob_info(_p(blob), blob.nbytes, _p(out))
    if st:
        raise ValueError(f"bad blob (status {st})")
    keys = ["codec", "n", "M", "O", "vmax", "tmax", "total_v", "total_tp", "total_t",
            "base_meshlet", "base_vtx", "base_tri", "max_record_bytes", "S", "n_out", "vw"]
    return Info({k: int(v) for k, v in zip(keys, out)})


class Encoded:
    """Result of the oracle encoder: blob bytes + source maps for round-trip checks."""

    def __init__(self, blob, src_vertex, src_tri, stats):
        self.blob = blob
        self.src_vertex = src_vertex      # (total_v,)  source vertex of each output vertex slot
        self.src_tri = src_tri            # (total_tp,) source triangle of each decoded slot, 0xFFFFFFFF = restart degenerate
        self.stats = dict(zip(["M", "total_v", "total_tp", "total_t", "restarts", "meshlets_built", "O"],
                              [int(x) for x in stats[:7]]))


def encode(mesh, vmax: int = 64, tmax: int = 126, codec: int = CODEC_REUSE, vw: bool = False) -> Encoded:
    """Oracle encoder (oracle.c ``or_encode``); ``vw``: per-meshlet attribute widths (FORMAT.md §1.4)."""
    idx = np.ascontiguousarray(mesh.indices, dtype=np.uint32).reshape(-1)
    attr = np.ascontiguousarray(mesh.attributes, dtype=np.float32)
    bits = np.asarray(mesh.bits, np.uint8)
    sem = np.asarray(mesh.semantic, np.uint8)
    obj = None if mesh.object_of_triangle is None else np.ascontiguousarray(mesh.object_of_triangle, np.uint32)
    bp, bn, sv, st = ctypes.c_void_p(), ctypes.c_uint64(), ctypes.c_void_p(), ctypes.c_void_p()
    stats = np.zeros(8, np.uint32)
    rc = lib().or_encode(_p(idx), mesh.num_triangles, _p(attr), mesh.num_vertices, mesh.n, _p(bits), _p(sem),
                         _p(obj), vmax, tmax, codec, 1 if vw else 0, ctypes.byref(bp), ctypes.byref(bn), ctypes.byref(sv),
                         ctypes.byref(st), _p(stats))
    if rc:
        raise ValueError(f"oracle encode failed: status {rc}")
    L = lib()
    blob = np.ctypeslib.as_array(ctypes.cast(bp, ctypes.POINTER(ctypes.c_uint8)), (bn.value,)).copy()
    tv, ttp = int(stats[1]), int(stats[2])
    srcv = np.ctypeslib.as_array(ctypes.cast(sv, ctypes.POINTER(ctypes.c_uint32)), (max(tv, 1),))[:tv].copy()
    srct = np.ctypeslib.as_array(ctypes.cast(st, ctypes.POINTER(ctypes.c_uint32)), (max(ttp, 1),))[:ttp].copy()
    L.or_free(bp)
    L.or_free(sv)
    L.or_free(st)
    return Encoded(blob, srcv, srct, stats)


def decode_meshlet(blob: np.ndarray, m: int, want_q=True, want_f=True):
    """Sequential decode of record m. Returns (err, meta, tri (T',3) local, q (V,n), f (V,n_out))."""
    info = blob_info(blob)
    tri = np.zeros(3 * 256, np.uint32)
    q = np.zeros(256 * 16, np.uint32) if want_q else None
    f = np.zeros(256 * 24, np.float32) if want_f else None
    meta = np.zeros(6, np.uint32)
    err = lib().or_decode_meshlet(_p(blob), blob.nbytes, m, _p(tri), _p(q), _p(f), _p(meta))
    V, Tp = int(meta[2]), int(meta[3])
    return (int(err), meta.astype(np.int64), tri[:3 * Tp].reshape(Tp, 3),
            None if q is None else q[:V * info.n].reshape(V, info.n),
            None if f is None else f[:V * info.n_out].reshape(V, info.n_out))


def decode(blob: np.ndarray, want_q=True, want_f=True, m0=0, m1=None):
    """Sequential decode of every record into whole-blob buffers (FORMAT.md §2, §4)."""
    info = blob_info(blob)
    m1 = info.M if m1 is None else m1
    idx = np.zeros(3 * info.total_tp, np.uint32)
    q = np.zeros(info.n * info.total_v, np.uint32) if want_q else None
    f = np.zeros(info.n_out * info.total_v, np.float32) if want_f else None
    err = np.zeros(max(m1 - m0, 1), np.uint32)
    allerr = lib().or_decode_range(_p(blob), blob.nbytes, m0, m1, _p(idx), _p(q), _p(f), _p(err))
    return int(allerr), err[:m1 - m0], idx, q, f


def decode_u8x4(blob: np.ndarray, m0=0, m1=None):
    """Local u8x4 index words (FORMAT.md §2) of the sequential decode: (err, words[total_tp])."""
    info = blob_info(blob)
    m1 = info.M if m1 is None else m1
    words = np.zeros(max(info.total_tp, 1), np.uint32)
    err = lib().or_decode_range_u8x4(_p(blob), blob.nbytes, m0, m1, _p(words))
    return int(err), words[:info.total_tp]


def decode_culled(blob: np.ndarray, view_dir, u8x4=False, want_q=True, want_f=True):
    """Cone-culled, compacted sequential decode (FORMAT.md §7).
    Returns (err, vis[M], counts {records, V, Tp, T}, idx, q, f) trimmed to the counts."""
    info = blob_info(blob)
    d = np.ascontiguousarray(np.asarray(view_dir, np.float32).reshape(3))
    idx = np.zeros(max((1 if u8x4 else 3) * info.total_tp, 1), np.uint32)
    q = np.zeros(max(info.n * info.total_v, 1), np.uint32) if want_q else None
    f = np.zeros(max(info.n_out * info.total_v, 1), np.float32) if want_f else None
    vis = np.zeros(max(info.M, 1), np.uint8)
    cnt = np.zeros(4, np.uint64)
    err = lib().or_decode_culled(_p(blob), blob.nbytes, _p(d), 1 if u8x4 else 0, _p(idx), _p(q), _p(f), _p(vis),
                                 _p(cnt))
    c = {"records": int(cnt[0]), "V": int(cnt[1]), "Tp": int(cnt[2]), "T": int(cnt[3])}
    return (int(err), vis[:info.M].astype(bool), c, idx[:(1 if u8x4 else 3) * c["Tp"]],
            None if q is None else q[:info.n * c["V"]], None if f is None else f[:info.n_out * c["V"]])


def add_cull(blob: np.ndarray, entries) -> np.ndarray:
    """Blob with the given cull table (FORMAT.md §1.5): entries (M, 4) = axis xyz, cutoff."""
    e = np.ascontiguousarray(np.asarray(entries, np.float32).reshape(-1))
    bp, bn = ctypes.c_void_p(), ctypes.c_uint64()
    rc = lib().or_add_cull(_p(blob), blob.nbytes, _p(e), ctypes.byref(bp), ctypes.byref(bn))
    if rc:
        raise ValueError(f"add_cull failed {rc}")
    out = np.ctypeslib.as_array(ctypes.cast(bp, ctypes.POINTER(ctypes.c_uint8)), (bn.value,)).copy()
    lib().or_free(bp)
    return out


def decode_range_raw(blob, m0, m1, idx, q, f):
    """Thread-friendly decode into caller buffers (ctypes releases the GIL)."""
    return lib().or_decode_range(_p(blob), blob.nbytes, m0, m1, _p(idx), _p(q), _p(f), None)


def checksum(words: np.ndarray, k0: int = 0) -> int:
    w = np.ascontiguousarray(words).view(np.uint32).reshape(-1)
    return int(lib().or_checksum(_p(w), w.size, k0))


def oct_decode(ex: float, ey: float):
    out = np.zeros(3, np.float32)
    lib().or_oct_decode(ctypes.c_float(ex), ctypes.c_float(ey), _p(out))
    return out


def pack(codec, bits, sem, delta, origin, vmax, tmax, V, Tp, R, obj, nbytes, L, lr, inc, byts, codes):
    """Serialise raw streams (no validation) — see oracle.c ``or_pack``."""
    n = len(bits)
    a32 = lambda x: np.ascontiguousarray(np.asarray(x, dtype=np.uint32).reshape(-1))
    a8 = lambda x: np.ascontiguousarray(np.asarray(x, dtype=np.uint8).reshape(-1))
    delta = np.ascontiguousarray(np.asarray(delta, np.float32).reshape(-1))
    origin = np.ascontiguousarray(np.asarray(origin, np.float32).reshape(-1))
    O = delta.size // n
    V, Tp, R, obj, nbytes, L = map(a32, (V, Tp, R, obj, nbytes, L))
    lr, inc, byts = a8(lr), a8(inc), a8(byts)
    codes = a32(codes)
    if byts.size == 0:
        byts = np.zeros(1, np.uint8)
    if codes.size == 0:
        codes = np.zeros(1, np.uint32)
    bp, bn = ctypes.c_void_p(), ctypes.c_uint64()
    rc = lib().or_pack(codec, n, _p(a8(bits)), _p(a8(sem)), O, _p(delta), _p(origin), vmax, tmax, V.size,
                       _p(V), _p(Tp), _p(R), _p(obj), _p(nbytes), _p(L), _p(lr), _p(inc), _p(byts), _p(codes),
                       ctypes.byref(bp), ctypes.byref(bn))
    if rc:
        raise ValueError(f"pack failed {rc}")
    blob = np.ctypeslib.as_array(ctypes.cast(bp, ctypes.POINTER(ctypes.c_uint8)), (bn.value,)).copy()
    lib().or_free(bp)
    return blob
