"""Seeded synthetic scenes shared by the oracle tests, the product tests and bench.py.

This module is *input generation only*: it builds triangle meshes and their float
attribute vectors (positions, normals, octahedral normal coordinates, texture
coordinates) with numpy.  It holds none of the method's arithmetic — no meshlet
building, no strips, no quantisation, no decoding — so that both the oracle
(``oracle/``) and the product (``paper_2404_06359_b200``) can consume the same
inputs without sharing any code (task rule ③).

Scene recipes follow SURVEY.md §8(d) and BASELINE.json ``configs``:

* cfg1 ``quad_grid(32, 32)``      2,048 tris, pos3+nrm3+uv2 (8 ch, ``P:476–478``)
* cfg2 ``torus(1000, 500)``       1,000,000 tris, pos3
* cfg3 ``displaced_sphere(913)``  ≈10.0M tris, pos3 + oct2 + uv2
* cfg4 ``city(...)``              ≈100M tris, instanced buildings (pos3 + oct2 + uv2)

Every attribute vector is float32; channel bit widths ``bits`` and ``semantic``
codes (FORMAT.md §1.1: 0 generic, 1 position, 2 normal, 3 texcoord, 4 oct) travel
with the mesh.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import os

import numpy as np

SEM_GENERIC, SEM_POSITION, SEM_NORMAL, SEM_TEXCOORD, SEM_OCT = 0, 1, 2, 3, 4


@dataclass
class Mesh:
    """An indexed triangle list (``P:208–211``) plus per-vertex attribute vectors."""

    indices: np.ndarray            # (T, 3) uint32, winding as authored
    attributes: np.ndarray         # (V, n) float32, vertex-major
    bits: list                     # n ints, b_c per channel
    semantic: list                 # n ints (SEM_*)
    object_of_triangle: np.ndarray | None = None   # (T,) uint32 or None
    name: str = "mesh"

    @property
    def num_vertices(self) -> int:
        return int(self.attributes.shape[0])

    @property
    def num_triangles(self) -> int:
        return int(self.indices.shape[0])

    @property
    def n(self) -> int:
        return int(self.attributes.shape[1])

    def with_bits(self, b) -> "Mesh":
        bits = [int(b)] * self.n if np.isscalar(b) else [int(x) for x in b]
        return Mesh(self.indices, self.attributes, bits, list(self.semantic),
                    self.object_of_triangle, self.name)


@dataclass
class InstancedScene:
    """Prototype meshes and instances (prototype id, translation) — cfg4."""

    prototypes: list
    instance_proto: np.ndarray     # (I,) uint32
    instance_offset: np.ndarray    # (I, 3) float32 translation of position channels
    name: str = "city"
    meta: dict = field(default_factory=dict)

    @property
    def num_triangles(self) -> int:
        return int(sum(self.prototypes[p].num_triangles for p in self.instance_proto))


# ----------------------------------------------------------------------------- helpers

def _grid_quads(nu: int, nv: int, wrap_u=False, wrap_v=False):
    """Triangulated (nu x nv)-quad grid; returns (T,3) indices over a (nu+1)x(nv+1) lattice
    (or nu x nv lattice per wrapped axis)."""
    cu = nu if wrap_u else nu + 1
    cv = nv if wrap_v else nv + 1
    i, j = np.meshgrid(np.arange(nu), np.arange(nv), indexing="ij")
    i1 = (i + 1) % cu
    j1 = (j + 1) % cv
    a = i * cv + j
    b = i1 * cv + j
    c = i1 * cv + j1
    d = i * cv + j1
    t0 = np.stack([a, b, c], -1).reshape(-1, 3)
    t1 = np.stack([a, c, d], -1).reshape(-1, 3)
    tris = np.empty((t0.shape[0] * 2, 3), dtype=np.int64)
    tris[0::2] = t0
    tris[1::2] = t1
    return tris.astype(np.uint32), cu, cv


def vertex_normals(pos: np.ndarray, tris: np.ndarray) -> np.ndarray:
    """Area-weighted vertex normals (float64 accumulate, unit length)."""
    p = pos.astype(np.float64)
    t = tris.astype(np.int64)
    fn = np.cross(p[t[:, 1]] - p[t[:, 0]], p[t[:, 2]] - p[t[:, 0]])
    vn = np.zeros_like(p)
    for k in range(3):
        for ax in range(3):
            vn[:, ax] += np.bincount(t[:, k], weights=fn[:, ax], minlength=p.shape[0])
    ln = np.linalg.norm(vn, axis=1, keepdims=True)
    ln[ln == 0] = 1.0
    return vn / ln


def oct_encode(nrm: np.ndarray) -> np.ndarray:
    """Unit vectors -> octahedral coordinates in [-1,1]^2 (Meyer et al. / Cigolle et al.,
    cited as prior work at ``P:244–245``).  Input preparation for the oct extension only."""
    n = nrm.astype(np.float64)
    s = np.abs(n).sum(axis=1, keepdims=True)
    s[s == 0] = 1.0
    p = n / s
    x, y, z = p[:, 0], p[:, 1], p[:, 2]
    sx = np.where(x >= 0, 1.0, -1.0)
    sy = np.where(y >= 0, 1.0, -1.0)
    ox = np.where(z < 0, (1.0 - np.abs(y)) * sx, x)
    oy = np.where(z < 0, (1.0 - np.abs(x)) * sy, y)
    return np.stack([ox, oy], 1)


def _value_noise(points: np.ndarray, seed: int, res: int = 12) -> np.ndarray:
    """Seeded trilinear lattice value noise in [-1, 1] on points in [-1, 1]^3."""
    rng = np.random.default_rng(seed)
    lat = rng.uniform(-1.0, 1.0, size=(res + 1,) * 3)
    u = (np.clip(points, -1.0, 1.0) + 1.0) * 0.5 * (res - 1e-9)
    i0 = np.floor(u).astype(np.int64)
    f = u - i0
    f = f * f * (3 - 2 * f)
    out = np.zeros(points.shape[0])
    for dx in (0, 1):
        wx = f[:, 0] if dx else 1 - f[:, 0]
        for dy in (0, 1):
            wy = f[:, 1] if dy else 1 - f[:, 1]
            for dz in (0, 1):
                wz = f[:, 2] if dz else 1 - f[:, 2]
                out += wx * wy * wz * lat[i0[:, 0] + dx, i0[:, 1] + dy, i0[:, 2] + dz]
    return out


def _cube_surface(k: int):
    """Subdivided unit-cube surface in [-1,1]^3, k x k quads per face, welded exactly on
    integer lattice coordinates.  Returns (points (V,3) float64, tris (T,3) uint32), CCW
    outward."""
    faces = []
    # (axis fixed, sign, u-axis, v-axis) chosen so (u x v) points along +sign*axis
    specs = [(0, +1, 1, 2), (0, -1, 2, 1), (1, +1, 2, 0), (1, -1, 0, 2), (2, +1, 0, 1), (2, -1, 1, 0)]
    keys = []
    for axis, sign, ua, va in specs:
        i, j = np.meshgrid(np.arange(k + 1), np.arange(k + 1), indexing="ij")
        lat = np.zeros((k + 1, k + 1, 3), dtype=np.int64)
        lat[..., axis] = k if sign > 0 else 0
        lat[..., ua] = i
        lat[..., va] = j
        keys.append(lat.reshape(-1, 3))
        tris, _, cv = _grid_quads(k, k)
        faces.append(tris.astype(np.int64))
    allkeys = np.concatenate(keys)
    code = (allkeys[:, 0] * (k + 1) + allkeys[:, 1]) * (k + 1) + allkeys[:, 2]
    uniq, inv = np.unique(code, return_inverse=True)
    off = 0
    tris = []
    for f in faces:
        tris.append(inv[f + off])
        off += (k + 1) ** 2
    tris = np.concatenate(tris)
    z = uniq % (k + 1)
    y = (uniq // (k + 1)) % (k + 1)
    x = uniq // ((k + 1) ** 2)
    pts = np.stack([x, y, z], 1).astype(np.float64) * (2.0 / k) - 1.0
    return pts, tris.astype(np.uint32)


# ----------------------------------------------------------------------------- scenes

def quad_grid(nx: int = 32, ny: int = 32, seed: int = 0, bits: int = 16) -> Mesh:
    """cfg1: nx*ny quads on [0,1]^2 (2*nx*ny tris), z = 0.05*sin(seeded phase),
    pos3 + nrm3 + uv2 (8 channels, the paper's example vector ``P:477``)."""
    rng = np.random.default_rng(seed)
    tris, cu, cv = _grid_quads(nx, ny)
    u, v = np.meshgrid(np.linspace(0, 1, cu), np.linspace(0, 1, cv), indexing="ij")
    u = u.reshape(-1)
    v = v.reshape(-1)
    ph = rng.uniform(0, 2 * np.pi, size=2)
    z = 0.05 * np.sin(6.0 * u + ph[0]) * np.sin(5.0 * v + ph[1])
    pos = np.stack([u, v, z], 1)
    nrm = vertex_normals(pos, tris)
    attr = np.concatenate([pos, nrm, np.stack([u, v], 1)], 1).astype(np.float32)
    return Mesh(tris, attr, [bits] * 8,
                [SEM_POSITION] * 3 + [SEM_NORMAL] * 3 + [SEM_TEXCOORD] * 2, None, f"grid{nx}x{ny}")


def torus(nu: int = 1000, nv: int = 500, R: float = 1.0, r: float = 0.4, bits: int = 16) -> Mesh:
    """cfg2: tessellated torus, nu*nv quads (2*nu*nv tris), positions only (3 ch)."""
    tris, cu, cv = _grid_quads(nu, nv, wrap_u=True, wrap_v=True)
    a, b = np.meshgrid(np.arange(cu) * (2 * np.pi / nu), np.arange(cv) * (2 * np.pi / nv), indexing="ij")
    a = a.reshape(-1)
    b = b.reshape(-1)
    pos = np.stack([(R + r * np.cos(b)) * np.cos(a), (R + r * np.cos(b)) * np.sin(a), r * np.sin(b)], 1)
    return Mesh(tris, pos.astype(np.float32), [bits] * 3, [SEM_POSITION] * 3, None, f"torus{nu}x{nv}")


def displaced_sphere(k: int = 913, seed: int = 0, amplitude: float = 0.02, bits: int = 16,
                     oct_normals: bool = True) -> Mesh:
    """cfg3: cube-sphere with 6*k*k quads (12*k^2 tris; k=913 -> 10.0M), radially displaced
    by seeded value noise (amplitude 2%), vertex normals -> octahedral (2 ch), spherical UVs.
    Channels: pos3 + oct2 + uv2 (7) — or pos3 + nrm3 + uv2 with ``oct_normals=False``."""
    pts, tris = _cube_surface(k)
    d = pts / np.linalg.norm(pts, axis=1, keepdims=True)
    disp = 1.0 + amplitude * _value_noise(d, seed)
    pos = d * disp[:, None]
    nrm = vertex_normals(pos, tris)
    uv = np.stack([np.arctan2(d[:, 1], d[:, 0]) / (2 * np.pi) + 0.5,
                   np.arccos(np.clip(d[:, 2], -1, 1)) / np.pi], 1)
    if oct_normals:
        attr = np.concatenate([pos, oct_encode(nrm), uv], 1).astype(np.float32)
        sem = [SEM_POSITION] * 3 + [SEM_OCT] * 2 + [SEM_TEXCOORD] * 2
    else:
        attr = np.concatenate([pos, nrm, uv], 1).astype(np.float32)
        sem = [SEM_POSITION] * 3 + [SEM_NORMAL] * 3 + [SEM_TEXCOORD] * 2
    return Mesh(tris, attr, [bits] * len(sem), sem, None, f"dsphere{k}")


def building(k: int, seed: int, bits: int = 16) -> Mesh:
    """One city building: subdivided box (12*k^2 tris), seeded footprint/height and a small
    seeded displacement, pos3 + oct2 + uv2."""
    rng = np.random.default_rng(seed)
    pts, tris = _cube_surface(k)
    w, dpt = rng.uniform(8.0, 20.0, size=2)
    h = rng.uniform(20.0, 120.0)
    scale = np.array([w * 0.5, dpt * 0.5, h * 0.5])
    pos = pts * scale + np.array([0.0, 0.0, h * 0.5])
    pos += 0.15 * _value_noise(pts, seed + 7919, res=8)[:, None] * pts
    nrm = vertex_normals(pos, tris)
    uv = np.stack([(pts[:, 0] + pts[:, 1]) * 0.25 + 0.5, (pts[:, 2] + 1.0) * 0.5], 1)
    attr = np.concatenate([pos, oct_encode(nrm), uv], 1).astype(np.float32)
    sem = [SEM_POSITION] * 3 + [SEM_OCT] * 2 + [SEM_TEXCOORD] * 2
    return Mesh(tris, attr, [bits] * 7, sem, None, f"building{seed}")


def city(num_instances: int = 1000, num_prototypes: int = 16, k: int = 91, seed: int = 0,
         bits: int = 16, k_jitter: int = 0) -> InstancedScene:
    """cfg4: instanced city — ``num_prototypes`` seeded buildings of 12*k_p^2 tris placed
    ``num_instances`` times on a jittered 2-D grid.  k_p = k (k=91 -> 99,372 tris) or, with
    k_jitter > 0, a seeded k_p in [k - k_jitter, k + k_jitter] per building (different
    subdivision, so different meshlet partitions and strips; mean ≈ 12 k^2 tris)."""
    rng = np.random.default_rng(seed)
    ks = [k] * num_prototypes if k_jitter <= 0 else \
        [int(x) for x in np.random.default_rng(seed + 77).integers(k - k_jitter, k + k_jitter + 1, num_prototypes)]
    if num_prototypes > 8:   # independent seeded meshes: build them on host threads
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(min(32, os.cpu_count() or 1)) as ex:
            protos = list(ex.map(lambda p: building(ks[p], seed * 1000 + p, bits), range(num_prototypes)))
    else:
        protos = [building(ks[p], seed * 1000 + p, bits) for p in range(num_prototypes)]
    side = int(np.ceil(np.sqrt(num_instances)))
    gi = np.arange(num_instances)
    gx, gy = gi % side, gi // side
    jitter = rng.uniform(-3.0, 3.0, size=(num_instances, 2))
    off = np.zeros((num_instances, 3), dtype=np.float32)
    off[:, 0] = gx * 32.0 + jitter[:, 0]
    off[:, 1] = gy * 32.0 + jitter[:, 1]
    proto = rng.integers(0, num_prototypes, size=num_instances).astype(np.uint32)
    return InstancedScene(protos, proto, off, f"city{num_instances}",
                          {"k": k, "k_jitter": k_jitter, "num_prototypes": num_prototypes, "seed": seed})


def random_patch(seed: int, nx: int = 12, ny: int = 9, drop: float = 0.15, n_ch: int = 5,
                 bits=None) -> Mesh:
    """Small irregular meshes for property tests: a jittered grid with a seeded fraction of
    triangles removed (holes, several components), shuffled triangle order, random
    rotation of each triangle's corner order, random per-channel bit widths."""
    rng = np.random.default_rng(seed)
    tris, cu, cv = _grid_quads(nx, ny)
    keep = rng.random(tris.shape[0]) >= drop
    tris = tris[keep]
    tris = tris[rng.permutation(tris.shape[0])]
    rot = rng.integers(0, 3, size=tris.shape[0])
    tris = np.stack([np.roll(t, -r) for t, r in zip(tris, rot)]) if tris.shape[0] else tris
    used = np.unique(tris)
    remap = np.full(cu * cv, -1, dtype=np.int64)
    perm = rng.permutation(used.shape[0])
    remap[used] = perm
    tris = remap[tris].astype(np.uint32)
    V = used.shape[0]
    attr = rng.normal(size=(V, n_ch)) * rng.uniform(0.1, 10.0, size=n_ch) + rng.uniform(-5, 5, size=n_ch)
    if bits is None:
        bits = [int(b) for b in rng.integers(3, 25, size=n_ch)]
    elif np.isscalar(bits):
        bits = [int(bits)] * n_ch
    return Mesh(tris, attr.astype(np.float32), list(bits), [SEM_GENERIC] * n_ch, None, f"patch{seed}")


def fan(n_tris: int, n_ch: int = 3, seed: int = 0) -> Mesh:
    """A single triangle fan around vertex 0 with ``n_tris`` triangles (long same-flag runs:
    the multi-word lookback case of ``P:444``)."""
    rng = np.random.default_rng(seed)
    tris = np.stack([np.zeros(n_tris, np.int64), np.arange(1, n_tris + 1), np.arange(2, n_tris + 2)], 1)
    ang = np.linspace(0, 1.9 * np.pi, n_tris + 1)
    pos = np.concatenate([[[0, 0, 0]], np.stack([np.cos(ang), np.sin(ang), 0 * ang], 1)])
    attr = pos[:, :n_ch] if n_ch <= 3 else np.concatenate([pos, rng.normal(size=(pos.shape[0], n_ch - 3))], 1)
    return Mesh(tris.astype(np.uint32), attr.astype(np.float32), [16] * n_ch,
                [SEM_POSITION] * min(3, n_ch) + [SEM_GENERIC] * max(0, n_ch - 3), None, f"fan{n_tris}")


def canonical_triangles(tris: np.ndarray) -> np.ndarray:
    """Rotate each oriented triangle so its smallest index comes first (cyclic rotation keeps
    winding), then sort rows — the multiset key of SPEC's round-trip invariant (``S:376``)."""
    t = np.asarray(tris, dtype=np.int64).reshape(-1, 3)
    if t.shape[0] == 0:
        return t
    r = np.argmin(t, axis=1)
    idx = (np.arange(3)[None, :] + r[:, None]) % 3
    c = np.take_along_axis(t, idx, axis=1)
    order = np.lexsort((c[:, 2], c[:, 1], c[:, 0]))
    return c[order]
