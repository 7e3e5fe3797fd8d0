"""Synthetic inputs of the named shapes — host-side, numpy.

None of these meshes is produced by the reference (it only subdivides by 4^s),
so they are generated here once and fed IDENTICALLY to the GPU path, the C
oracle and the compiled reference. Conventions follow the reference:

* counter RNG ``splitmix64`` / ``hash_combine`` / ``Rng`` (rng.hpp:9-36);
* edges in ``build_adjacency`` order (mesh.cpp:27-63): sorted by (v0 < v1),
  f0 the lower incident face, f1 = -1 on boundary edges;
* spherical UVs as ``assign_spherical_uvs`` (mesh.cpp:352-369);
* the blob displacement field of ``make_blob`` (mesh.cpp:307-330);
* cameras from ``sample_views_on_sphere`` (camera.cpp:61-77) + ``look_at``
  (camera.cpp:10-23);
* targets from a perturbed copy (positions x1.05 about the centroid, diffuse
  +0.08), as ``cmd_gradcheck`` builds them (gradcheck.cpp:49-73).

Textures are quantised to fp32-representable doubles so the device may keep
them as fp32 with no loss.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import numpy as np

_M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15


# ---------------------------------------------------------------- RNG (rng.hpp)
def splitmix64(x):
    """Vectorised splitmix64 over uint64 arrays (rng.hpp:9-14)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = x + np.uint64(GOLDEN)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


def hash_combine(a, b):
    """rng.hpp:16-18."""
    a = np.asarray(a, dtype=np.uint64)
    b = np.asarray(b, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return splitmix64(a ^ (b + np.uint64(GOLDEN) + (a << np.uint64(6)) + (a >> np.uint64(2))))


class Rng:
    """Vectorised ``collodiff::Rng`` (rng.hpp:20-50): one stream per key tuple."""

    def __init__(self, seed, *keys):
        h = np.asarray(seed, dtype=np.uint64)
        for k in keys:
            h = hash_combine(h, k)
        self.state = splitmix64(h)

    def next_u64(self):
        self.state = splitmix64(self.state)
        return self.state

    def next_double(self):
        return (self.next_u64() >> np.uint64(11)).astype(np.float64) * 2.0 ** -53

    def next_gaussian(self):
        u1 = float(self.next_double())
        u2 = float(self.next_double())
        if u1 < 1e-300:
            u1 = 1e-300
        return math.sqrt(-2.0 * math.log(u1)) * math.cos(6.283185307179586 * u2)


# ---------------------------------------------------------------- data classes
@dataclass
class Camera:
    """camera.hpp:12-23."""
    origin: np.ndarray
    right: np.ndarray
    up: np.ndarray
    forward: np.ndarray
    fov_deg: float
    width: int
    height: int


@dataclass
class Mesh:
    positions: np.ndarray  # V x 3 f64
    triangles: np.ndarray  # T x 3 i32
    uvs: np.ndarray        # V x 2 f64
    edges: np.ndarray = None  # E x 4 i32 (v0, v1, f0, f1)

    def __post_init__(self):
        self.positions = np.ascontiguousarray(self.positions, dtype=np.float64)
        self.triangles = np.ascontiguousarray(self.triangles, dtype=np.int32)
        self.uvs = np.ascontiguousarray(self.uvs, dtype=np.float64)
        if self.edges is None:
            self.edges = build_adjacency(self.triangles, len(self.positions))

    @property
    def V(self):
        return len(self.positions)

    @property
    def T(self):
        return len(self.triangles)

    @property
    def E(self):
        return len(self.edges)


@dataclass
class Scene:
    """scene.hpp:17-23 (maps as H x W x C arrays)."""
    mesh: Mesh
    diffuse: np.ndarray    # H x W x 3
    specular: np.ndarray   # H x W x 3
    roughness: np.ndarray  # H x W
    cameras: list
    light: np.ndarray = field(default_factory=lambda: np.array([20.0, 20.0, 20.0]))
    background: np.ndarray = field(default_factory=lambda: np.zeros(3))

    @property
    def tex_res(self):
        return self.diffuse.shape[1], self.diffuse.shape[0]


# ---------------------------------------------------------------- adjacency
def build_adjacency(tris, nv):
    """Edge list in the reference's std::map order (mesh.cpp:27-63)."""
    tris = np.asarray(tris, dtype=np.int64)
    nt = len(tris)
    if nt == 0:
        return np.zeros((0, 4), dtype=np.int32)
    a = tris[:, [0, 1, 2]].reshape(-1)
    b = tris[:, [1, 2, 0]].reshape(-1)
    f = np.repeat(np.arange(nt, dtype=np.int64), 3)
    lo = np.minimum(a, b)
    hi = np.maximum(a, b)
    key = lo * nv + hi
    order = np.lexsort((f, key))
    key, f = key[order], f[order]
    starts = np.flatnonzero(np.r_[True, key[1:] != key[:-1]])
    counts = np.diff(np.r_[starts, len(key)])
    if counts.max() > 2:
        raise ValueError("non-manifold edge")
    e = np.empty((len(starts), 4), dtype=np.int32)
    e[:, 0] = key[starts] // nv
    e[:, 1] = key[starts] % nv
    e[:, 2] = f[starts]
    second = np.where(counts > 1, starts + 1, starts)
    e[:, 3] = np.where(counts > 1, f[second], -1)
    return e


# ---------------------------------------------------------------- meshes
def _icosahedron():
    t = (1.0 + math.sqrt(5.0)) / 2.0
    p = np.array([[-1, t, 0], [1, t, 0], [-1, -t, 0], [1, -t, 0], [0, -1, t], [0, 1, t],
                  [0, -1, -t], [0, 1, -t], [t, 0, -1], [t, 0, 1], [-t, 0, -1], [-t, 0, 1]],
                 dtype=np.float64)
    p /= np.linalg.norm(p, axis=1, keepdims=True)
    f = [[0, 11, 5], [0, 5, 1], [0, 1, 7], [0, 7, 10], [0, 10, 11], [1, 5, 9], [5, 11, 4],
         [11, 10, 2], [10, 7, 6], [7, 1, 8], [3, 9, 4], [3, 4, 2], [3, 2, 6], [3, 6, 8],
         [3, 8, 9], [4, 9, 5], [2, 4, 11], [6, 2, 10], [8, 6, 7], [9, 8, 1]]
    return p, np.array(f, dtype=np.int64)


def geodesic_sphere(freq: int, radius: float = 0.5) -> Mesh:
    """Class-I geodesic sphere: each icosahedron face split into freq^2 triangles.

    V = 10 f^2 + 2, T = 20 f^2, E = 30 f^2 (f = 11: 1,212 / 2,420 / 3,630;
    f = 59: 34,812 / 69,620 / 104,430 — SURVEY.md §8(d)). Outward CCW winding.
    """
    base, faces = _icosahedron()
    index = {}
    pos = []

    def vid(key_parts):
        key = tuple(sorted((int(v), int(w)) for v, w in key_parts if w != 0))
        i = index.get(key)
        if i is None:
            i = len(pos)
            index[key] = i
            p = np.zeros(3)
            for v, w in key:
                p = p + base[v] * (w / freq)
            pos.append(p / np.linalg.norm(p))
        return i

    tris = []
    for (A, B, C) in faces:
        grid = {}
        for i in range(freq + 1):
            for j in range(freq + 1 - i):
                grid[(i, j)] = vid([(A, freq - i - j), (B, i), (C, j)])
        for i in range(freq):
            for j in range(freq - i):
                tris.append((grid[(i, j)], grid[(i + 1, j)], grid[(i, j + 1)]))
                if i + j + 1 < freq:
                    tris.append((grid[(i + 1, j)], grid[(i + 1, j + 1)], grid[(i, j + 1)]))
    pos = np.array(pos) * radius
    tris = np.array(tris, dtype=np.int64)
    # orient outward (the icosahedron's faces are CCW from outside)
    n = np.cross(pos[tris[:, 1]] - pos[tris[:, 0]], pos[tris[:, 2]] - pos[tris[:, 0]])
    flip = (n * pos[tris].mean(axis=1)).sum(axis=1) < 0
    tris[flip] = tris[flip][:, [0, 2, 1]]
    return Mesh(pos, tris.astype(np.int32), spherical_uvs(pos))


def icosphere(subdivisions: int, radius: float = 0.5) -> Mesh:
    """make_icosphere (mesh.cpp:270-298): 4^s midpoint subdivision, vertices in
    creation order — the mesh the reference's own tests render."""
    base, faces = _icosahedron()
    pos = [base[i] for i in range(12)]
    tris = [tuple(int(x) for x in f) for f in faces]
    for _ in range(subdivisions):
        mids = {}

        def mid(a, b):
            key = (min(a, b), max(a, b))
            i = mids.get(key)
            if i is None:
                p = pos[a] + pos[b]
                pos.append(p / math.sqrt(float(p[0] * p[0] + p[1] * p[1] + p[2] * p[2])))
                i = mids[key] = len(pos) - 1
            return i
        nxt = []
        for a, b, c in tris:
            ab, bc, ca = mid(a, b), mid(b, c), mid(c, a)
            nxt += [(a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca)]
        tris = nxt
    P = np.array(pos) * radius
    return Mesh(P, np.array(tris, np.int32), spherical_uvs(P))


def spherical_uvs(pos):
    """assign_spherical_uvs (mesh.cpp:352-369)."""
    c = pos.sum(axis=0) / max(1, len(pos))
    d = pos - c
    ln = np.sqrt((d * d).sum(axis=1))
    uv = np.full((len(pos), 2), 0.5)
    ok = ln >= 1e-12
    dd = d[ok] / ln[ok, None]
    u = 0.5 + np.arctan2(dd[:, 1], dd[:, 0]) / 6.283185307179586
    v = 0.5 - np.arcsin(np.clip(dd[:, 2], -1.0, 1.0)) / 3.141592653589793
    uv[ok, 0] = np.clip(u, 0.0, 1.0)
    uv[ok, 1] = np.clip(v, 0.0, 1.0)
    return uv


def blob(freq: int, seed: int = 5, amplitude: float = 0.15) -> Mesh:
    """``make_blob``'s displacement field (mesh.cpp:307-330) on a geodesic sphere."""
    m = geodesic_sphere(freq, 0.5)
    rng = Rng(seed, 0xB10B)
    lobes = []
    for _ in range(5):
        d = np.array([rng.next_gaussian(), rng.next_gaussian(), rng.next_gaussian()])
        d = d / math.sqrt(float(d @ d))
        freq_l = 1.0 + 2.0 * float(rng.next_double())
        amp = amplitude * (0.4 + 0.6 * float(rng.next_double()))
        phase = 6.2831853 * float(rng.next_double())
        lobes.append((d, freq_l, amp, phase))
    p = m.positions
    dirs = p / np.sqrt((p * p).sum(axis=1))[:, None]
    r = np.full(len(p), 0.5)
    for d, fr, amp, ph in lobes:
        r = r + amp * np.cos(fr * 3.1415926 * (dirs @ d) + ph) * 0.5
    pos = dirs * r[:, None]
    return Mesh(pos, m.triangles, spherical_uvs(pos))


def torus_knot(n_seg: int = 1000, n_ring: int = 100, p: int = 2, q: int = 3,
               tube: float = 0.04) -> Mesh:
    """(p, q) torus-knot tube, 2 * n_seg * n_ring triangles, genus-1 closed
    manifold; fits the unit box. UV = (curve parameter, ring angle)."""
    phi = np.arange(n_seg) * (2.0 * math.pi / n_seg)

    def curve(f):
        r = 2.0 + np.cos(q * f)
        return np.stack([r * np.cos(p * f), r * np.sin(p * f), -np.sin(q * f)], axis=-1)

    c = curve(phi)
    h = 1e-4
    tng = curve(phi + h) - curve(phi - h)
    tng /= np.linalg.norm(tng, axis=1, keepdims=True)
    acc = curve(phi + h) - 2 * c + curve(phi - h)
    nrm = acc - (acc * tng).sum(axis=1, keepdims=True) * tng
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    bin_ = np.cross(tng, nrm)
    scale = 1.0 / 6.0  # curve extent ~[-3, 3] -> unit box
    th = np.arange(n_ring) * (2.0 * math.pi / n_ring)
    ring = (np.cos(th)[None, :, None] * nrm[:, None, :] + np.sin(th)[None, :, None] * bin_[:, None, :])
    pos = (c[:, None, :] * scale + tube * ring).reshape(-1, 3)
    i = np.arange(n_seg)[:, None]
    j = np.arange(n_ring)[None, :]
    a = i * n_ring + j
    b = ((i + 1) % n_seg) * n_ring + j
    c2 = ((i + 1) % n_seg) * n_ring + (j + 1) % n_ring
    d = i * n_ring + (j + 1) % n_ring
    tris = np.concatenate([np.stack([a, b, c2], -1).reshape(-1, 3),
                           np.stack([a, c2, d], -1).reshape(-1, 3)]).astype(np.int64)
    # orient outward from the tube centre line
    cen = np.repeat(c * scale, n_ring, axis=0)
    fn = np.cross(pos[tris[:, 1]] - pos[tris[:, 0]], pos[tris[:, 2]] - pos[tris[:, 0]])
    out = pos[tris].mean(axis=1) - cen[tris[:, 0]]
    flip = (fn * out).sum(axis=1) < 0
    tris[flip] = tris[flip][:, [0, 2, 1]]
    uv = np.stack([np.repeat(np.arange(n_seg) / n_seg, n_ring),
                   np.tile(np.arange(n_ring) / n_ring, n_seg)], axis=-1)
    return Mesh(pos, tris.astype(np.int32), uv)


# ---------------------------------------------------------------- cameras
def _normalize(v):
    v = np.asarray(v, dtype=np.float64)
    ln = math.sqrt(float(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]))
    return v / ln


def _cross(a, b):
    return np.array([a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]])


def look_at(origin, target, up_hint, fov_deg, width, height) -> Camera:
    """Camera::look_at (camera.cpp:10-23)."""
    origin = np.asarray(origin, dtype=np.float64)
    fwd = _normalize(np.asarray(target, dtype=np.float64) - origin)
    hint = np.asarray(up_hint, dtype=np.float64)
    c = _cross(fwd, hint)
    if math.sqrt(float(c[0] * c[0] + c[1] * c[1] + c[2] * c[2])) < 1e-6:
        hint = np.array([1.0, 0.0, 0.0])
    right = _normalize(_cross(fwd, hint))
    up = _cross(right, fwd)
    return Camera(origin, right, up, fwd, float(fov_deg), int(width), int(height))


def sample_views_on_sphere(count, radius, seed, fov_deg=45.0, width=64, height=64):
    """camera.cpp:61-77."""
    if count < 1:
        raise ValueError("view count must be >= 1")
    rng = Rng(seed, 0xF1B0)
    phase = float(rng.next_double()) * 6.283185307179586
    golden_angle = 2.399963229728653
    cams = []
    for i in range(count):
        z = 0.3 if count == 1 else 1.0 - 2.0 * (i + 0.5) / count
        r = math.sqrt(max(0.0, 1.0 - z * z))
        phi = golden_angle * i + phase
        pos = np.array([radius * r * math.cos(phi), radius * r * math.sin(phi), radius * z])
        cams.append(look_at(pos, [0, 0, 0], [0, 0, 1], fov_deg, width, height))
    return cams


# ---------------------------------------------------------------- textures
def random_maps(res: int, seed: int = 7):
    """Per-texel diffuse U(0.2,0.8)^3, specular U(0.02,0.2)^3, roughness
    U(0.1,0.9) from Rng(seed, 0x7e0+map, texel), quantised to fp32."""
    idx = np.arange(res * res, dtype=np.uint64)

    def draws(map_id, lo, hi, ch):
        rng = Rng(seed, 0x7E0 + map_id, idx)
        cols = [lo + (hi - lo) * rng.next_double() for _ in range(ch)]
        a = np.stack(cols, axis=-1) if ch > 1 else cols[0]
        return a.astype(np.float32).astype(np.float64)

    d = draws(1, 0.2, 0.8, 3).reshape(res, res, 3)
    s = draws(2, 0.02, 0.2, 3).reshape(res, res, 3)
    r = draws(3, 0.1, 0.9, 1).reshape(res, res)
    return d, s, r


def constant_maps(res, diffuse, specular, roughness):
    """make_constant_maps (material.cpp:5-12)."""
    d = np.broadcast_to(np.asarray(diffuse, dtype=np.float64), (res, res, 3)).copy()
    s = np.broadcast_to(np.asarray(specular, dtype=np.float64), (res, res, 3)).copy()
    r = np.full((res, res), float(roughness))
    return d, s, r


# ---------------------------------------------------------------- configs
CONFIGS = {
    # name: (mesh builder, tex res, views, image, spp)
    "cfg1": (lambda: geodesic_sphere(11), 128, 4, 128, 4),
    "cfg2": (lambda: blob(59), 512, 50, 512, 16),
    "cfg3": (lambda: blob(59), 1024, 100, 512, 16),
    "cfg4": (lambda: torus_knot(), 1024, 64, 1024, 16),
}


def make_scene(mesh: Mesh, tex_res: int, n_views: int, image: int, seed: int = 7,
               fov: float = 40.0, radius: float = 2.5, view_seed: int = 11) -> Scene:
    d, s, r = random_maps(tex_res, seed)
    cams = sample_views_on_sphere(n_views, radius, view_seed, fov, image, image)
    return Scene(mesh, d, s, r, cams)


def config_scene(name: str, n_views: int | None = None) -> tuple[Scene, int]:
    build, tex, views, image, spp = CONFIGS[name]
    return make_scene(build(), tex, views if n_views is None else n_views, image), spp


def perturbed_target_scene(scene: Scene) -> Scene:
    """gradcheck.cpp:49-56: positions x1.05 about the centroid, diffuse +0.08."""
    p = scene.mesh.positions
    c = p.sum(axis=0) / len(p)
    pos = c + (p - c) * 1.05
    m = Mesh(pos, scene.mesh.triangles, scene.mesh.uvs, scene.mesh.edges)
    diff = np.clip(scene.diffuse + 0.08, 0.0, 1.0).astype(np.float32).astype(np.float64)
    return replace(scene, mesh=m, diffuse=diff)


def camera_struct_array(cams):
    """Pack cameras as cdr_camera records (include/cdr.h)."""
    dt = np.dtype([("origin", "<f8", 3), ("right", "<f8", 3), ("up", "<f8", 3),
                   ("forward", "<f8", 3), ("fov_deg", "<f8"), ("width", "<i4"),
                   ("height", "<i4")])
    a = np.zeros(len(cams), dtype=dt)
    for i, c in enumerate(cams):
        a[i] = (c.origin, c.right, c.up, c.forward, c.fov_deg, c.width, c.height)
    return a


CAMERA_DTYPE = camera_struct_array([]).dtype
