"""The reference's own known-answer and property tests (proj/tests/*.cpp),
restated against both implementations: the CPU oracle (always) and the GPU
path (marked gpu). Each test cites the reference test it mirrors."""
import math

import numpy as np
import pytest

from paper_2103_15208_b200 import scenes as S
from tests import backends

KINDS = ["oracle", pytest.param("gpu", marks=pytest.mark.gpu)]
PI = 3.14159265358979323846


def quad(center, span_u, span_v):
    """make_quad (mesh.cpp:332-340)."""
    c, u, v = map(lambda a: np.asarray(a, dtype=np.float64), (center, span_u, span_v))
    pos = np.array([c - u * 0.5 - v * 0.5, c + u * 0.5 - v * 0.5, c + u * 0.5 + v * 0.5, c - u * 0.5 + v * 0.5])
    return S.Mesh(pos, np.array([[0, 1, 2], [0, 2, 3]], np.int32), np.array([[0, 0], [1, 0], [1, 1], [0, 1]], float))


def plane_scene(dist, albedo, light, span=10.0, image=16, fov=45.0):
    """lambertian_plane_scene (tests/support/test_scenes.hpp:72-83)."""
    m = quad([0, 0, dist], [0, span, 0], [span, 0, 0])
    d, s, r = S.constant_maps(4, albedo, (0, 0, 0), 0.5)
    cam = S.look_at([0, 0, 0], [0, 0, dist], [0, 1, 0], fov, image, image)
    sc = S.Scene(m, d, s, r, [cam])
    sc.light = np.asarray(light, dtype=np.float64)
    return sc


def sphere_scene(subdiv, views, image):
    """sphere_scene (test_scenes.hpp:92-102)."""
    m = S.icosphere(subdiv, 0.5)
    d, s, r = S.constant_maps(8, (0.55, 0.4, 0.3), (0.05, 0.05, 0.05), 0.4)
    return S.Scene(m, d, s, r, S.sample_views_on_sphere(views, 2.5, 11, 40.0, image, image))


def plane_radiance(albedo, light, dist, d):
    dz = d[2]
    return 0.0 if dz <= 0 else light * albedo * (dz ** 3 / (PI * dist * dist))


@pytest.mark.parametrize("kind", KINDS)
def test_radiance_plane_inverse_square(kind):
    # test_render.cpp:13-23
    for dist in (1.0, 2.0):
        b = backends.make(kind, plane_scene(dist, (1, 1, 1), (PI, PI, PI)))
        rad, _ = b.radiance_at(0, [8.0, 8.0])
        assert rad[0, 0] == pytest.approx(1.0 / dist ** 2, rel=1e-9)
        assert rad[0, 1] == pytest.approx(1.0 / dist ** 2, rel=1e-9)


@pytest.mark.parametrize("kind", KINDS)
def test_miss_returns_background(kind):
    # test_render.cpp:25-32
    sc = plane_scene(1.0, (1, 1, 1), (1, 1, 1), span=0.01)
    sc.background = np.array([0.1, 0.2, 0.3])
    b = backends.make(kind, sc)
    rad, tri = b.radiance_at(0, [1.0, 1.0])
    assert tri[0] == -1
    assert rad[0, 0] == pytest.approx(0.1) and rad[0, 2] == pytest.approx(0.3)


@pytest.mark.parametrize("kind", KINDS)
def test_render_matches_quadrature_within_3_sigma(kind):
    # test_render.cpp:34-65
    albedo, light = 0.8, PI
    sc = plane_scene(1.0, (albedo,) * 3, (light,) * 3)
    b = backends.make(kind, sc)
    img, mask, _ = b.render(0, 64, 5)
    cam = sc.cameras[0]
    th = math.tan(cam.fov_deg * PI / 360.0)
    q = 16
    for y in range(16):
        for x in range(16):
            vals = []
            for j in range(q):
                for i in range(q):
                    px, py = x + (i + 0.5) / q, y + (j + 0.5) / q
                    sx = (2.0 * px / 16 - 1.0) * th
                    sy = (1.0 - 2.0 * py / 16) * th
                    d = cam.forward + cam.right * sx + cam.up * sy
                    d = d / np.linalg.norm(d)
                    vals.append(plane_radiance(albedo, light, 1.0, d))
            vals = np.array(vals)
            sigma = math.sqrt(max(0.0, (vals ** 2).mean() - vals.mean() ** 2) / 64)
            assert abs(img[y, x, 0] - vals.mean()) <= 3 * sigma + 1e-6
            assert mask[y, x] == 1.0


@pytest.mark.parametrize("kind", KINDS)
def test_doubling_spp_halves_variance(kind):
    # test_render.cpp:78-115
    sc = sphere_scene(2, 1, 16)
    b = backends.make(kind, sc)
    _, mask, _ = b.render(0, 16, 0)
    cand = np.argwhere((mask > 0.2) & (mask < 0.8))
    assert len(cand)
    py, px = cand[0]

    def var(spp):
        v = np.array([b.render(0, spp, 1000 + i)[0][py, px, 0] for i in range(48)])
        return (v ** 2).mean() - v.mean() ** 2
    # The reference test doubles 8 -> 16 spp, but 16 = 4x4 switches on jittered
    # stratification (render.cpp:15-20): the reference library itself measures
    # a ratio of 0.0385 on this scene, so test_render.cpp:114 fails as shipped.
    # The Monte Carlo property is pinned on a non-square pair instead (the
    # reference gives 0.42 for 6 -> 12), and stratification must only help.
    v6, v12 = var(6), var(12)
    assert v6 > 0
    assert v12 / v6 == pytest.approx(0.5, rel=0.45)
    assert var(16) < 0.5 * var(8)


@pytest.mark.parametrize("kind", KINDS)
def test_render_deterministic(kind):
    # test_render.cpp:117-127
    b = backends.make(kind, sphere_scene(2, 1, 24))
    a1, m1, h1 = b.render(0, 8, 42)
    a2, m2, h2 = b.render(0, 8, 42)
    np.testing.assert_array_equal(a1, a2)
    np.testing.assert_array_equal(h1, h2)


@pytest.mark.parametrize("kind", KINDS)
def test_silhouette_single_triangle_and_coplanar_quad(kind):
    # test_silhouette.cpp:30-47
    m = S.Mesh(np.array([[-0.3, -0.3, 2], [0.3, -0.3, 2], [0, 0.4, 2]], float), np.array([[0, 1, 2]], np.int32),
               np.array([[0, 0], [1, 0], [0, 1]], float))
    d, s, r = S.constant_maps(4, (0.5,) * 3, (0,) * 3, 0.5)
    cam = S.look_at([0, 0, 0], [0, 0, 1], [0, 1, 0], 45, 32, 32)
    segs, _ = backends.make(kind, S.Scene(m, d, s, r, [cam])).silhouettes(0)
    assert len(segs) == 3 and (segs["length_px"] > 0).all()
    cam = S.look_at([0, 0, 0], [0, 0, 2], [0, 1, 0], 45, 32, 32)
    segs, _ = backends.make(kind, S.Scene(quad([0, 0, 2], [0.6, 0, 0], [0, 0.6, 0]), d, s, r, [cam])).silhouettes(0)
    assert len(segs) == 4


@pytest.mark.parametrize("kind", KINDS)
def test_silhouette_predicate_oracle_and_great_circle(kind):
    # test_silhouette.cpp:49-67
    m = S.icosphere(2, 0.5)
    d, s, r = S.constant_maps(4, (0.5,) * 3, (0,) * 3, 0.5)
    cam = S.look_at([0, 0, 3], [0, 0, 0], [0, 1, 0], 40, 64, 64)
    segs, _ = backends.make(kind, S.Scene(m, d, s, r, [cam])).silhouettes(0)
    P, T = m.positions, m.triangles
    fn = np.cross(P[T[:, 1]] - P[T[:, 0]], P[T[:, 2]] - P[T[:, 0]])
    expected = set()
    for v0, v1, f0, f1 in m.edges:
        dd = (P[v0] + P[v1]) * 0.5 - cam.origin
        if f1 < 0 or np.sign(fn[f0] @ dd) != np.sign(fn[f1] @ dd):
            expected.add((v0, v1))
    assert {(a, b) for a, b in zip(segs["v0"], segs["v1"])} == expected
    mid = (segs["p0"] + segs["p1"]) * 0.5
    assert (np.abs(mid[:, 2]) < 0.2).all()


@pytest.mark.parametrize("kind", KINDS)
def test_silhouette_behind_camera_and_clipping(kind):
    # test_silhouette.cpp:69-83
    m = S.icosphere(1, 0.5)
    d, s, r = S.constant_maps(4, (0.5,) * 3, (0,) * 3, 0.5)
    away = S.look_at([0, 0, 2], [0, 0, 5], [0, 1, 0], 45, 32, 32)
    segs, _ = backends.make(kind, S.Scene(m, d, s, r, [away])).silhouettes(0)
    assert len(segs) == 0
    close = S.look_at([0, 0, 0.8], [0, 0, 0], [0, 1, 0], 45, 32, 32)
    segs, _ = backends.make(kind, S.Scene(m, d, s, r, [close])).silhouettes(0)
    for q in (segs["q0"], segs["q1"]):
        assert (q >= -1e-9).all() and (q <= 32 + 1e-9).all()


@pytest.mark.parametrize("kind", KINDS)
def test_silhouette_2d_to_3d_projective(kind):
    # test_silhouette.cpp:85-101
    m = S.icosphere(2, 0.5)
    d, s, r = S.constant_maps(4, (0.5,) * 3, (0,) * 3, 0.5)
    cam = S.look_at([0.4, 0.2, 2.5], [0, 0, 0], [0, 1, 0], 40, 64, 64)
    segs, _ = backends.make(kind, S.Scene(m, d, s, r, [cam])).silhouettes(0)
    assert len(segs)
    th = math.tan(40 * PI / 360.0)
    for sg in segs[:8]:
        for u in (0.25, 0.5, 0.75):
            w0, w1 = (1 - u) / sg["z0"], u / sg["z1"]
            t = (w0 * sg["t0"] + w1 * sg["t1"]) / (w0 + w1)
            p = sg["p0"] + (sg["p1"] - sg["p0"]) * t
            v = p - cam.origin
            z = v @ cam.forward
            q = np.array([((v @ cam.right) / (z * th) + 1) * 32, (1 - (v @ cam.up) / (z * th)) * 32])
            expect = sg["q0"] + (sg["q1"] - sg["q0"]) * u
            assert np.linalg.norm(q - expect) < 1e-6


@pytest.mark.parametrize("kind", KINDS)
def test_laplacian_properties(kind):
    # test_laplacian.cpp:41-88
    m = S.icosphere(2, 0.5)
    d, s, r = S.constant_maps(4, (0.5,) * 3, (0,) * 3, 0.5)
    b = backends.make(kind, S.Scene(m, d, s, r, S.sample_views_on_sphere(1, 2.5, 11)))
    for mode in (0, 1):
        outer, inner, vals = b.laplacian(mode)
        A = np.zeros((m.V, m.V))
        for j in range(m.V):
            A[inner[outer[j]:outer[j + 1]], j] = vals[outer[j]:outer[j + 1]]
        assert np.abs(A.sum(axis=1)).max() < 1e-9
        assert np.abs(A - A.T).max() < 1e-12
    # uniform tetrahedron by hand (make_tetrahedron, mesh.cpp:342-350)
    sc = 0.5 / math.sqrt(3.0)
    P = np.array([[sc, sc, sc], [sc, -sc, -sc], [-sc, sc, -sc], [-sc, -sc, sc]])
    tet = S.Mesh(P, np.array([[0, 2, 1], [0, 1, 3], [0, 3, 2], [1, 2, 3]], np.int32), np.zeros((4, 2)))
    b = backends.make(kind, S.Scene(tet, d, s, r, S.sample_views_on_sphere(1, 2.5, 11)))
    outer, inner, vals = b.laplacian(1)
    LV = backends.csc_times(outer, inner, vals, P)
    for i in range(4):
        np.testing.assert_allclose(LV[i], sum(P[j] - P[i] for j in range(4) if j != i), rtol=1e-12, atol=1e-15)
    # degenerate weights stay finite and clamped
    Pd = np.array([[0, 0, 0], [1, 0, 0], [0.5, 1e-13, 0], [0.5, -1, 0]], float)
    dm = S.Mesh(Pd, np.array([[0, 1, 2], [1, 0, 3]], np.int32), np.zeros((4, 2)))
    b = backends.make(kind, S.Scene(dm, d, s, r, S.sample_views_on_sphere(1, 2.5, 11)))
    _, _, vals = b.laplacian(0)
    assert np.isfinite(vals).all() and (np.abs(vals) <= 4e4 + 1).all()


def test_equilateral_patch_harmonic():
    # test_laplacian.cpp:51-60: planar interior vertices are harmonic
    from oracle.pyoracle import Oracle
    n = 6
    pts = [(i + 0.5 * j, j * math.sqrt(3) / 2, 0.0) for j in range(n) for i in range(n)]
    tris = []
    for j in range(n - 1):
        for i in range(n - 1):
            a, b, c, d = j * n + i, j * n + i + 1, (j + 1) * n + i, (j + 1) * n + i + 1
            tris += [(a, b, c), (b, d, c)]
    m = S.Mesh(np.array(pts), np.array(tris, np.int32), np.zeros((n * n, 2)))
    dd, ss, rr = S.constant_maps(4, (0.5,) * 3, (0,) * 3, 0.5)
    o = Oracle(S.Scene(m, dd, ss, rr, S.sample_views_on_sphere(1, 2.5, 11)))
    boundary = set(m.edges[m.edges[:, 3] < 0][:, :2].ravel())
    for mode in (0, 1):
        _, _, (outer, inner, vals) = o.laplacian(mode)
        LV = backends.csc_times(outer, inner, vals, m.positions)
        for v in range(m.V):
            if v not in boundary:
                assert np.abs(LV[v]).max() < 1e-6
