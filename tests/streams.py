"""Test-side helpers: hand-written streams, a tiny FORMAT.md record reader, and an
independent pure-Python strip encoder for brute-force path-cover checks.

None of this is used by the product or by the oracle; it exists to pin both.
"""
from __future__ import annotations

import itertools

import numpy as np


def read_records(blob: np.ndarray):
    """Minimal FORMAT.md §1 reader: yields dicts of record header fields + section words."""
    b = blob.view(np.uint8)
    u32 = lambda off: int(np.frombuffer(b[off:off + 4].tobytes(), "<u4")[0])
    u64 = lambda off: int(np.frombuffer(b[off:off + 8].tobytes(), "<u8")[0])
    codec, n, M = u32(8), u32(12), u32(16)
    vw = u32(60) & 1                                   # per-meshlet widths (FORMAT.md §1.4)
    off_dir, off_rec = u64(64), u64(80)
    hdr = (16 + 4 * n + (n if vw else 0) + 15) // 16 * 16
    out = []
    for m in range(M):
        r0 = off_rec + 16 * u32(off_dir + 4 * m)
        V, Tp = int(b[r0 + 8]) + 1, int(b[r0 + 9]) + 1
        W = 0 if codec == 3 else (Tp + 31) // 32     # Basic records have no flag words
        lr = np.frombuffer(b[r0 + hdr:r0 + hdr + 4 * W].tobytes(), "<u4")
        inc = np.frombuffer(b[r0 + hdr + 4 * W:r0 + hdr + 8 * W].tobytes(), "<u4") if codec == 2 else None
        out.append(dict(vtx_base=u32(r0), tri_base=u32(r0 + 4), V=V, Tp=Tp,
                        object=int(b[r0 + 10]) | (int(b[r0 + 11]) << 8),
                        R=int(b[r0 + 12]) | (int(b[r0 + 13]) << 8),
                        L=[u32(r0 + 16 + 4 * c) for c in range(n)], lr=lr, inc=inc, codec=codec,
                        basic=(b[r0 + hdr:r0 + hdr + 3 * Tp].copy() if codec == 3 else None),
                        widths=([int(x) for x in b[r0 + 16 + 4 * n:r0 + 16 + 5 * n]] if vw
                                else [int(x) for x in b[96:96 + n]]),
                        size=16 * (u32(off_dir + 4 * m + 4) - u32(off_dir + 4 * m)), offset=r0, hdr=hdr))
    return out


def gts_meshlet(V, flags, idx):
    """One GTS record's raw fields: flags[t] (t=1..T'-1, 1=R), idx[t-1]."""
    Tp = len(flags) + 1
    return dict(V=V, Tp=Tp, lr=[0] + list(flags), inc=[0] * Tp, bytes=list(idx))


def basic_meshlet(V, tris):
    """One Basic record's raw fields: a local triangle list."""
    flat = [int(x) for t in tris for x in t]
    return dict(V=V, Tp=len(tris), lr=[0] * len(tris), inc=[0] * len(tris), bytes=flat)


def reuse_meshlet(V, flags, inc, reuse):
    Tp = len(flags) + 1
    return dict(V=V, Tp=Tp, lr=[0] + list(flags), inc=[0] + list(inc), bytes=list(reuse))


def pack_meshlets(orc, codec, meshlets, n=1, bits=(8,), sem=None, codes=None, L=None,
                  delta=None, origin=None, vmax=256, tmax=256, R=None, obj=None):
    """Pack a list of raw meshlet dicts with the oracle's un-validating packer."""
    M = len(meshlets)
    sem = [0] * n if sem is None else sem
    V = [m["V"] for m in meshlets]
    Tp = [m["Tp"] for m in meshlets]
    lr = list(itertools.chain.from_iterable(m["lr"] for m in meshlets))
    inc = list(itertools.chain.from_iterable(m["inc"] for m in meshlets))
    byts = list(itertools.chain.from_iterable(m["bytes"] for m in meshlets))
    nbytes = [len(m["bytes"]) for m in meshlets]
    if codes is None:
        codes = np.zeros(sum(V) * n, np.uint32)
    if L is None:
        L = np.zeros(M * n, np.uint32)
    delta = np.ones(n, np.float32) if delta is None else delta
    origin = np.zeros(n, np.float32) if origin is None else origin
    R = [0] * M if R is None else R
    obj = [0] * M if obj is None else obj
    return orc.pack(codec, list(bits), sem, delta, origin, vmax, tmax, V, Tp, R, obj, nbytes, L,
                    lr, inc, byts, codes)


def closed_form_decode(flags, N):
    """The data-parallel closed form (FORMAT.md §2): each triangle on its own,
    j(t) = max{k<t : f_k != f_t} with f_0 = L, written independently of the oracle."""
    f = [0] + list(flags)
    out = [(N[0], N[1], N[2])]
    for t in range(1, len(f)):
        j = -1
        for k in range(t - 1, -1, -1):
            if f[k] != f[t]:
                j = k
                break
        if f[t]:
            out.append((N[t + 1], N[j + 1], N[t + 2]))
        else:
            out.append((N[j + 1], N[t + 1], N[t + 2]))
    return out


def py_strip_encode(tris, paths):
    """Independent pure-Python GTS encoder for one meshlet given a path cover.

    tris: list of oriented source triangles (tuples of source vertex ids);
    paths: list of lists of triangle positions (each consecutive pair edge-adjacent).
    Returns (V, flags, N_local, src_of_local) following the paper's edge rule
    (continue across the right edge (b,c) or the left edge (c,a)), the
    4-degenerate restart (pattern S:350) and ascending relabel."""
    steps = []  # (flag, vertex)
    cur = None
    for pi, path in enumerate(paths):
        t0 = tris[path[0]]
        k = 0
        if len(path) > 1:
            # keep the authored rotation when the successor already lies across (b,c) or
            # (c,a), i.e. the unshared vertex is a or b; otherwise rotate once
            nxt = set(tris[path[1]])
            if [i for i in range(3) if t0[i] not in nxt][0] == 2:
                k = 1
        p, q, r = t0[k], t0[(k + 1) % 3], t0[(k + 2) % 3]
        if cur is None:
            N = [p, q, r]
        else:
            a, b, c = cur
            for fl, w in ((1, c), (0, q), (0, q), (1, p), (1, r)):
                steps.append((fl, w))
        cur = (p, q, r)
        for ti in path[1:]:
            a, b, c = cur
            tv = tris[ti]
            if b in tv and c in tv:
                w = [x for x in tv if x not in (b, c)][0]
                steps.append((1, w))
                cur = (c, b, w)
            elif a in tv and c in tv:
                w = [x for x in tv if x not in (a, c)][0]
                steps.append((0, w))
                cur = (a, c, w)
            else:
                raise ValueError("path not edge-connected through the exit edges")
    seq = N + [w for _, w in steps]
    order = {}
    for v in seq:
        order.setdefault(v, len(order))
    Nl = [order[v] for v in seq]
    src = [v for v, _ in sorted(order.items(), key=lambda kv: kv[1])]
    return len(order), [fl for fl, _ in steps], Nl, src


def reuse_fields(N_local):
    """Increment flags + reuse buffer from a local step sequence."""
    inc, reuse, mx = [], [], 2
    for w in N_local[3:]:
        if w == mx + 1:
            inc.append(1)
            mx = w
        else:
            inc.append(0)
            reuse.append(w)
    return inc, reuse
