"""B200-native meshlet decompression (arXiv 2404.06359) — thin Python binding of libmc.so.

Every step of the hot path runs in the C-ABI library (``include/mc.h``): the host
encoder in C++, the decoder in hand-written sm_100a CUDA.  This module only marshals
arguments (numpy host arrays, torch device tensors, CUDA stream handles).  There is
no Python or CPU fallback: if ``libmc.so`` is missing, importing the binding fails.

Function names follow the C ABI: ``mc_encode``, ``mc_decode_meshlets``,
``mc_decode_stats``, ``mc_decode_host``, ``mc_blob_instance``, ...
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _build

# MC_LIB: another build of the same library (tests/test_gpu_bounds.py loads the
# bounds-checking build in a subprocess); default the in-tree product build
LIB_PATH = os.environ.get("MC_LIB", _build.LIB)

MC_CODEC_GTS, MC_CODEC_GTS_REUSE, MC_CODEC_BASIC = 1, 2, 3
MC_DECODE_BLOB_LOCAL_INDICES, MC_DECODE_INDEX_LOCAL_U8X4 = 1, 2
MC_ENCODE_VARIABLE_WIDTHS, MC_ENCODE_CULL_CONES = 1, 2
ABI_VERSION = 4
MC_DECODE_WORK_WORDS = 256
MC_DERR_RECORD, MC_DERR_COUNTS, MC_DERR_INDEX, MC_DERR_REUSE, MC_DERR_OBJECT = 1, 2, 4, 8, 16


class MCError(RuntimeError):
    pass


class mc_layout(ctypes.Structure):
    _fields_ = [(k, ctypes.c_uint32) for k in
                ("codec", "n", "n_out", "S", "num_meshlets", "num_objects", "v_max", "t_max",
                 "total_v", "total_tp", "total_t", "base_meshlet", "base_vtx", "base_tri", "max_record_bytes")] + \
               [("off_dir", ctypes.c_uint64), ("off_obj", ctypes.c_uint64), ("off_rec", ctypes.c_uint64),
                ("total_bytes", ctypes.c_uint64), ("bits", ctypes.c_uint8 * 16), ("semantic", ctypes.c_uint8 * 16),
                ("flags", ctypes.c_uint32), ("off_cull", ctypes.c_uint64)]


class mc_mesh(ctypes.Structure):
    _fields_ = [("num_vertices", ctypes.c_uint32), ("num_triangles", ctypes.c_uint32),
                ("indices", ctypes.c_void_p), ("attributes", ctypes.c_void_p),
                ("num_channels", ctypes.c_uint32), ("bits", ctypes.c_void_p), ("semantic", ctypes.c_void_p),
                ("object_of_triangle", ctypes.c_void_p)]


class mc_encode_params(ctypes.Structure):
    _fields_ = [("max_vertices", ctypes.c_uint32), ("max_triangles", ctypes.c_uint32),
                ("codec", ctypes.c_uint32), ("num_threads", ctypes.c_uint32), ("flags", ctypes.c_uint32)]


class mc_decode_args(ctypes.Structure):
    _fields_ = [("layout", ctypes.POINTER(mc_layout)), ("d_blob", ctypes.c_void_p),
                ("first", ctypes.c_uint32), ("count", ctypes.c_uint32),
                ("d_indices", ctypes.c_void_p), ("d_vertices", ctypes.c_void_p),
                ("d_quantized", ctypes.c_void_p), ("flags", ctypes.c_uint32), ("d_work", ctypes.c_void_p)]


class mc_host_decode_args(ctypes.Structure):
    _fields_ = [("layout", ctypes.POINTER(mc_layout)), ("h_blob", ctypes.c_void_p), ("d_blob", ctypes.c_void_p),
                ("h_indices", ctypes.c_void_p), ("h_vertices", ctypes.c_void_p), ("h_quantized", ctypes.c_void_p),
                ("d_indices", ctypes.c_void_p), ("d_vertices", ctypes.c_void_p), ("d_quantized", ctypes.c_void_p),
                ("flags", ctypes.c_uint32), ("chunks", ctypes.c_uint32)]


class mc_stats(ctypes.Structure):
    _fields_ = [(k, ctypes.c_uint64) for k in
                ("checksum_indices", "checksum_vertices", "checksum_quantized", "triangles", "degenerate",
                 "vertices", "multiword_lookbacks")] + \
               [(k, ctypes.c_uint32) for k in ("max_lookback", "error_bits", "first_bad_meshlet", "num_bad")]


class mc_info(ctypes.Structure):
    _fields_ = [(k, ctypes.c_uint32) for k in ("codec", "n", "num_meshlets", "num_objects")] + \
               [(k, ctypes.c_uint64) for k in
                ("total_v", "total_tp", "total_t", "restarts", "header_bytes", "directory_bytes", "object_bytes",
                 "cull_bytes", "record_bytes", "total_bytes", "record_header_bytes", "flag_bytes", "index_bytes",
                 "attribute_bytes", "padding_bytes")] + \
               [("bits_per_triangle", ctypes.c_double), ("index_bits_per_triangle", ctypes.c_double)]


class mc_channel_grid(ctypes.Structure):
    _fields_ = [("delta", ctypes.c_float), ("origin", ctypes.c_float), ("bits", ctypes.c_uint32),
                ("w_steps", ctypes.c_uint32), ("W_steps", ctypes.c_uint64), ("w", ctypes.c_double),
                ("W", ctypes.c_double), ("info_bits", ctypes.c_double)]


STATS_BYTES = ctypes.sizeof(mc_stats)
EXPORTS = ["mc_encode", "mc_blob_instance", "mc_blob_instance_range", "mc_blob_from_bytes", "mc_blob_bytes", "mc_blob_source_map",
           "mc_blob_encode_stats", "mc_blob_free", "mc_parse_header", "mc_blob_shard_ranges", "mc_blob_extract",
           "mc_decode_meshlets", "mc_decode_stats", "mc_stats_reset", "mc_decode_host", "mc_status_str",
           "mc_abi_version", "mc_decode_culled", "mc_decode_culled_scratch_bytes", "mc_blob_info"]

_lib = None


def lib() -> ctypes.CDLL:
    """Load libmc.so (built in-tree by ``__graft_entry__.build()``); fail loudly if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        P, u32, sz = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_size_t
        for name in EXPORTS:
            getattr(L, name).restype = ctypes.c_int
        L.mc_status_str.restype = ctypes.c_char_p
        L.mc_abi_version.restype = u32
        if L.mc_abi_version() != ABI_VERSION:
            raise ImportError(f"{LIB_PATH}: ABI {L.mc_abi_version()} != {ABI_VERSION}; rebuild with __graft_entry__.build()")
        L.mc_encode.argtypes = [ctypes.POINTER(mc_mesh), ctypes.POINTER(mc_encode_params), ctypes.POINTER(P)]
        L.mc_blob_instance.argtypes = [P, u32, P, P, u32, ctypes.POINTER(P)]
        L.mc_blob_instance_range.argtypes = [P, u32, P, P, u32, u32, u32, ctypes.POINTER(P)]
        L.mc_blob_from_bytes.argtypes = [P, sz, ctypes.POINTER(P)]
        L.mc_blob_bytes.argtypes = [P, ctypes.POINTER(P), ctypes.POINTER(sz)]
        L.mc_blob_source_map.argtypes = [P, ctypes.POINTER(P), ctypes.POINTER(P)]
        L.mc_blob_encode_stats.argtypes = [P, ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64)]
        L.mc_blob_free.argtypes = [P]
        L.mc_blob_free.restype = None
        L.mc_parse_header.argtypes = [P, sz, ctypes.POINTER(mc_layout)]
        L.mc_blob_shard_ranges.argtypes = [P, sz, u32, P, P]
        L.mc_blob_extract.argtypes = [P, sz, u32, u32, ctypes.POINTER(P)]
        L.mc_decode_meshlets.argtypes = [ctypes.POINTER(mc_decode_args), P]
        L.mc_decode_stats.argtypes = [ctypes.POINTER(mc_decode_args), P, P]
        L.mc_stats_reset.argtypes = [P, P]
        L.mc_decode_host.argtypes = [ctypes.POINTER(mc_host_decode_args), P]
        L.mc_status_str.argtypes = [ctypes.c_int]
        L.mc_decode_culled.argtypes = [ctypes.POINTER(mc_decode_args), P, P, sz, P, P, P]
        L.mc_decode_culled_scratch_bytes.argtypes = [ctypes.POINTER(mc_layout)]
        L.mc_decode_culled_scratch_bytes.restype = sz
        L.mc_blob_info.argtypes = [P, sz, ctypes.POINTER(mc_info), P, u32]
        _lib = L
    return _lib


def _check(rc: int, what: str):
    if rc != 0:
        raise MCError(f"{what}: {lib().mc_status_str(rc).decode()} (status {rc})")


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


# ----------------------------------------------------------------------------- blobs

class _Handle:
    """Owns one mc_blob; freed when the last Blob or byte view referencing it dies."""

    def __init__(self, h: ctypes.c_void_p):
        self.h = h

    def __del__(self):
        if self.h is not None and _lib is not None:
            _lib.mc_blob_free(self.h)
            self.h = None


class _View:
    """numpy __array_interface__ over the blob's bytes that keeps its _Handle alive."""

    def __init__(self, handle: _Handle, ptr: int, n: int):
        self.handle = handle
        self.__array_interface__ = {"shape": (n,), "typestr": "|u1", "data": (ptr, True), "version": 3}


class Blob:
    """An encoded meshlet stream (FORMAT.md) owned by libmc (``mc_blob``)."""

    def __init__(self, handle: ctypes.c_void_p):
        self._owner = _Handle(handle)
        self._h = handle
        bp, n = ctypes.c_void_p(), ctypes.c_size_t()
        _check(lib().mc_blob_bytes(self._h, ctypes.byref(bp), ctypes.byref(n)), "mc_blob_bytes")
        # read-only view; it keeps the library object alive even after this Blob is gone
        self.bytes = np.asarray(_View(self._owner, bp.value or 0, n.value))
        self.layout = parse_header(self.bytes)

    @classmethod
    def from_bytes(cls, data: np.ndarray) -> "Blob":
        data = np.ascontiguousarray(data, dtype=np.uint8)
        h = ctypes.c_void_p()
        _check(lib().mc_blob_from_bytes(_p(data), data.nbytes, ctypes.byref(h)), "mc_blob_from_bytes")
        return cls(h)

    def source_map(self):
        sv, st = ctypes.c_void_p(), ctypes.c_void_p()
        _check(lib().mc_blob_source_map(self._h, ctypes.byref(sv), ctypes.byref(st)), "mc_blob_source_map")
        L = self.layout
        v = np.ctypeslib.as_array(ctypes.cast(sv, ctypes.POINTER(ctypes.c_uint32)), (max(L.total_v, 1),))[:L.total_v]
        t = np.ctypeslib.as_array(ctypes.cast(st, ctypes.POINTER(ctypes.c_uint32)), (max(L.total_tp, 1),))[:L.total_tp]
        return v.copy(), t.copy()

    def encode_stats(self):
        r, s = ctypes.c_uint64(), ctypes.c_uint64()
        _check(lib().mc_blob_encode_stats(self._h, ctypes.byref(r), ctypes.byref(s)), "mc_blob_encode_stats")
        return {"restarts": r.value, "split_meshlets": s.value}

    def shard_ranges(self, parts: int):
        return mc_blob_shard_ranges(self.bytes, parts)

    def extract(self, first: int, count: int) -> "Blob":
        return mc_blob_extract(self.bytes, first, count)

    def info(self, grids: bool = True):
        return mc_blob_info(self.bytes, grids)


def parse_header(data: np.ndarray) -> mc_layout:
    L = mc_layout()
    _check(lib().mc_parse_header(_p(data), data.nbytes, ctypes.byref(L)), "mc_parse_header")
    return L


def mc_encode(mesh, max_vertices: int = 64, max_triangles: int = 126, codec: int = MC_CODEC_GTS_REUSE,
              num_threads: int = 0, variable_widths: bool = False, cull_cones: bool = False) -> Blob:
    """Encode a mesh (any object with indices/attributes/bits/semantic[/object_of_triangle]);
    ``variable_widths``: per-meshlet attribute code widths (MC_ENCODE_VARIABLE_WIDTHS)."""
    idx = np.ascontiguousarray(mesh.indices, dtype=np.uint32)
    attr = np.ascontiguousarray(mesh.attributes, dtype=np.float32)
    bits = np.ascontiguousarray(np.asarray(mesh.bits, dtype=np.uint8))
    sem = np.ascontiguousarray(np.asarray(mesh.semantic, dtype=np.uint8))
    obj = getattr(mesh, "object_of_triangle", None)
    obj = None if obj is None else np.ascontiguousarray(obj, dtype=np.uint32)
    m = mc_mesh(attr.shape[0], idx.reshape(-1, 3).shape[0], _p(idx), _p(attr), attr.shape[1], _p(bits), _p(sem),
                _p(obj))
    prm = mc_encode_params(max_vertices, max_triangles, codec, num_threads,
                           (MC_ENCODE_VARIABLE_WIDTHS if variable_widths else 0) |
                           (MC_ENCODE_CULL_CONES if cull_cones else 0))
    h = ctypes.c_void_p()
    _check(lib().mc_encode(ctypes.byref(m), ctypes.byref(prm), ctypes.byref(h)), "mc_encode")
    return Blob(h)


def mc_blob_instance(protos, proto_of_instance, offsets) -> Blob:
    arr = (ctypes.c_void_p * len(protos))(*[p._h.value for p in protos])
    pi = np.ascontiguousarray(proto_of_instance, dtype=np.uint32)
    off = np.ascontiguousarray(offsets, dtype=np.float32).reshape(-1)
    h = ctypes.c_void_p()
    _check(lib().mc_blob_instance(ctypes.cast(arr, ctypes.c_void_p), len(protos), _p(pi), _p(off), pi.size,
                                  ctypes.byref(h)), "mc_blob_instance")
    return Blob(h)


def mc_blob_instance_range(protos, proto_of_instance, offsets, first_instance: int, instance_count: int) -> Blob:
    arr = (ctypes.c_void_p * len(protos))(*[p._h.value for p in protos])
    pi = np.ascontiguousarray(proto_of_instance, dtype=np.uint32)
    off = np.ascontiguousarray(offsets, dtype=np.float32).reshape(-1)
    h = ctypes.c_void_p()
    _check(lib().mc_blob_instance_range(ctypes.cast(arr, ctypes.c_void_p), len(protos), _p(pi), _p(off), pi.size,
                                        first_instance, instance_count, ctypes.byref(h)), "mc_blob_instance_range")
    return Blob(h)


def mc_blob_shard_ranges(data: np.ndarray, parts: int):
    first = np.zeros(parts, np.uint32)
    count = np.zeros(parts, np.uint32)
    _check(lib().mc_blob_shard_ranges(_p(data), data.nbytes, parts, _p(first), _p(count)), "mc_blob_shard_ranges")
    return [(int(f), int(c)) for f, c in zip(first, count)]


def mc_blob_info(data: np.ndarray, grids: bool = True):
    """Blob summary (dict of mc_info) and, with `grids`, the per-object per-channel grids
    (list over objects of lists over channels of dicts of mc_channel_grid)."""
    data = np.ascontiguousarray(data, dtype=np.uint8)
    L = parse_header(data)
    info = mc_info()
    arr = (mc_channel_grid * max(1, L.num_objects * L.n))() if grids else None
    _check(lib().mc_blob_info(_p(data), data.nbytes, ctypes.byref(info),
                              ctypes.cast(arr, ctypes.c_void_p) if grids else None,
                              L.num_objects * L.n if grids else 0), "mc_blob_info")
    d = {k: getattr(info, k) for k, _ in mc_info._fields_}
    if not grids:
        return d, None
    g = [[{k: getattr(arr[o * L.n + c], k) for k, _ in mc_channel_grid._fields_} for c in range(L.n)]
         for o in range(L.num_objects)]
    return d, g


def mc_blob_extract(data: np.ndarray, first: int, count: int) -> Blob:
    h = ctypes.c_void_p()
    _check(lib().mc_blob_extract(_p(data), data.nbytes, first, count, ctypes.byref(h)), "mc_blob_extract")
    return Blob(h)


# ----------------------------------------------------------------------------- device decode

def _tptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream_handle(stream):
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _check_sizes(layout: mc_layout, d_blob, d_indices, d_vertices, d_quantized, flags: int):
    """Refuse device buffers smaller than mc.h states (the C ABI takes raw pointers)."""
    L = layout
    need = {"d_blob": (d_blob, L.total_bytes, 1),
            "d_indices": (d_indices, (1 if flags & MC_DECODE_INDEX_LOCAL_U8X4 else 3) * L.total_tp, 4),
            "d_vertices": (d_vertices, L.n_out * L.total_v, 4), "d_quantized": (d_quantized, L.n * L.total_v, 4)}
    for name, (t, n, esz) in need.items():
        if t is not None and t.numel() * t.element_size() < n * esz:
            raise MCError(f"{name}: {t.numel() * t.element_size()} bytes < {n * esz} required")


def _device_of(t):
    """torch.cuda.device guard for the tensor's device (the C ABI runs on the current device)."""
    import torch
    return torch.cuda.device(t.device)


def _check_work(d_work):
    if d_work is not None and d_work.numel() * d_work.element_size() < 4 * MC_DECODE_WORK_WORDS:
        raise MCError(f"d_work: {d_work.numel() * d_work.element_size()} bytes < {4 * MC_DECODE_WORK_WORDS} required")


def _args(layout, d_blob, d_indices, d_vertices, d_quantized, first, count, flags, d_work):
    _check_sizes(layout, d_blob, d_indices, d_vertices, d_quantized, flags)
    _check_work(d_work)
    count = layout.num_meshlets - first if count is None else count
    return mc_decode_args(ctypes.pointer(layout), d_blob.data_ptr(), first, count, d_indices.data_ptr(),
                          None if d_vertices is None else d_vertices.data_ptr(),
                          None if d_quantized is None else d_quantized.data_ptr(), flags,
                          None if d_work is None else d_work.data_ptr())


def mc_decode_meshlets(layout: mc_layout, d_blob, d_indices, d_vertices=None, d_quantized=None, first: int = 0,
                       count: int | None = None, flags: int = 0, stream=None, d_work=None):
    """Enqueue the decode of records [first, first+count) on `stream` (torch stream or None);
    d_work: optional zero-initialised int32 tensor of MC_DECODE_WORK_WORDS (include/mc.h)."""
    a = _args(layout, d_blob, d_indices, d_vertices, d_quantized, first, count, flags, d_work)
    with _device_of(d_blob):
        _check(lib().mc_decode_meshlets(ctypes.byref(a), _stream_handle(stream)), "mc_decode_meshlets")


def mc_stats_reset(d_stats, stream=None):
    with _device_of(d_stats):
        _check(lib().mc_stats_reset(_tptr(d_stats), _stream_handle(stream)), "mc_stats_reset")


def mc_decode_stats(layout: mc_layout, d_blob, d_indices, d_stats, d_vertices=None, d_quantized=None, first: int = 0,
                    count: int | None = None, flags: int = 0, stream=None, d_work=None):
    a = _args(layout, d_blob, d_indices, d_vertices, d_quantized, first, count, flags, d_work)
    with _device_of(d_blob):
        _check(lib().mc_decode_stats(ctypes.byref(a), _tptr(d_stats), _stream_handle(stream)), "mc_decode_stats")


def read_stats(d_stats) -> dict:
    """Copy a device mc_stats (a uint8 tensor of STATS_BYTES) to a dict (synchronises)."""
    raw = d_stats.cpu().numpy().tobytes()
    s = mc_stats.from_buffer_copy(raw)
    return {k: getattr(s, k) for k, _ in mc_stats._fields_}


def mc_decode_host(layout: mc_layout, h_blob, d_blob, h_indices, d_indices, h_vertices=None, d_vertices=None,
                   h_quantized=None, d_quantized=None, flags: int = 0, stream=None, chunks: int = 32):
    """End-to-end decode from host tensors (pinned for overlap): H2D, decode, D2H ordered on
    `stream`; chunks >= 2 pipelines them over byte-balanced record ranges (include/mc.h)."""
    _check_sizes(layout, d_blob, d_indices, d_vertices, d_quantized, flags)
    _check_sizes(layout, h_blob, h_indices, h_vertices, h_quantized, flags)
    a = mc_host_decode_args(ctypes.pointer(layout), h_blob.data_ptr(), d_blob.data_ptr(), h_indices.data_ptr(),
                            None if h_vertices is None else h_vertices.data_ptr(),
                            None if h_quantized is None else h_quantized.data_ptr(), d_indices.data_ptr(),
                            None if d_vertices is None else d_vertices.data_ptr(),
                            None if d_quantized is None else d_quantized.data_ptr(), flags, chunks)
    with _device_of(d_blob):
        _check(lib().mc_decode_host(ctypes.byref(a), _stream_handle(stream)), "mc_decode_host")


class DeviceBlob:
    """A blob resident in HBM plus output buffers sized from its layout (torch tensors)."""

    def __init__(self, blob, device="cuda", want_vertices=True, want_quantized=False, index_format="u32"):
        """index_format: "u32" = three global u32 indices per triangle (FORMAT.md §2),
        "u8x4" = one word of meshlet-local u8 indices per triangle (MC_DECODE_INDEX_LOCAL_U8X4)."""
        import torch
        if index_format not in ("u32", "u8x4"):
            raise ValueError(index_format)
        data = blob.bytes if isinstance(blob, Blob) else np.ascontiguousarray(blob, dtype=np.uint8)
        self.layout = parse_header(data)
        L = self.layout
        self.index_format = index_format
        self.index_flags = MC_DECODE_INDEX_LOCAL_U8X4 if index_format == "u8x4" else 0
        self.d_blob = torch.from_numpy(np.array(data, copy=True)).to(device)
        self.indices = torch.empty((1 if self.index_flags else 3) * L.total_tp, dtype=torch.int32, device=device)
        self.vertices = torch.empty(L.n_out * L.total_v, dtype=torch.float32, device=device) if want_vertices else None
        self.quantized = torch.empty(L.n * L.total_v, dtype=torch.int32, device=device) if want_quantized else None
        self.stats = torch.zeros(STATS_BYTES, dtype=torch.uint8, device=device)
        # claim-counter work buffer (include/mc.h d_work): zeroed once, left zeroed by every
        # completed decode; decodes of this DeviceBlob must be ordered on one stream
        self.work = torch.zeros(MC_DECODE_WORK_WORDS, dtype=torch.int32, device=device)

    def decode(self, stream=None, flags=0, first=0, count=None):
        mc_decode_meshlets(self.layout, self.d_blob, self.indices, self.vertices, self.quantized, first, count,
                           flags | self.index_flags, stream, d_work=self.work)

    def decode_stats(self, stream=None, flags=0, first=0, count=None) -> dict:
        mc_stats_reset(self.stats, stream)
        mc_decode_stats(self.layout, self.d_blob, self.indices, self.stats, self.vertices, self.quantized, first,
                        count, flags | self.index_flags, stream, d_work=self.work)
        return read_stats(self.stats)

    def decode_culled(self, view_dir, stream=None, flags=0, stats=False):
        """Enqueue the cone-culled compacted decode (FORMAT.md §7) for a unit view direction;
        counts land in ``self.cull_counts`` (device int32[4]: records, V, T', T)."""
        import torch
        L = self.layout
        if getattr(self, "cull_scratch", None) is None:
            nb = lib().mc_decode_culled_scratch_bytes(ctypes.byref(L))
            # zero once: every completed culled decode leaves its look-back flags zero (mc.h)
            self.cull_scratch = torch.zeros((nb + 15) // 16 * 16, dtype=torch.uint8, device=self.d_blob.device)
            self.cull_counts = torch.zeros(4, dtype=torch.int32, device=self.d_blob.device)
        _check_sizes(L, self.d_blob, self.indices, self.vertices, self.quantized, flags | self.index_flags)
        a = mc_decode_args(ctypes.pointer(L), self.d_blob.data_ptr(), 0, L.num_meshlets, self.indices.data_ptr(),
                           None if self.vertices is None else self.vertices.data_ptr(),
                           None if self.quantized is None else self.quantized.data_ptr(), flags | self.index_flags,
                           self.work.data_ptr())
        d = (ctypes.c_float * 3)(*[float(x) for x in view_dir])
        if stats:
            mc_stats_reset(self.stats, stream)
        with _device_of(self.d_blob):
            _check(lib().mc_decode_culled(ctypes.byref(a), ctypes.cast(d, ctypes.c_void_p),
                                          self.cull_scratch.data_ptr(), self.cull_scratch.numel(),
                                          self.cull_counts.data_ptr(), self.stats.data_ptr() if stats else None,
                                          _stream_handle(stream)), "mc_decode_culled")
        return read_stats(self.stats) if stats else None

    def read_cull_counts(self) -> dict:
        c = self.cull_counts.cpu().numpy().view(np.uint32)
        return {"records": int(c[0]), "V": int(c[1]), "Tp": int(c[2]), "T": int(c[3])}

    def algorithmic_bytes(self) -> int:
        """Compressed bytes read (directory + records + object table) + decompressed bytes written."""
        L = self.layout
        read = (L.total_bytes - L.off_rec) + 4 * (L.num_meshlets + 1) + 8 * L.n * L.num_objects
        write = (4 if self.index_flags else 12) * L.total_tp + (4 * L.n_out * L.total_v if self.vertices is not None else 0) + \
            (4 * L.n * L.total_v if self.quantized is not None else 0)
        return int(read + write)
