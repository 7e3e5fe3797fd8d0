"""Pin the C restatement (oracle/cdr_oracle.c) against the reference library
compiled from its own unmodified sources (oracle/_ref). CPU only.

Single-threaded reference runs are deterministic, so every comparison here is
bit-exact (the oracle replicates the reference's operation order and is built
with -ffp-contract=off like the reference build).
"""
import ctypes as C

import numpy as np
import pytest

from oracle import pyoracle
from oracle.pyoracle import Oracle, RefLib, cdr_camera, layout_for, settings
from paper_2103_15208_b200 import scenes as S
from tests.scenes_util import blob_scene, small_scene, targets_for

pytestmark = pytest.mark.ref

D = C.POINTER(C.c_double)


def dp(a):
    return np.ascontiguousarray(a, dtype=np.float64).ctypes.data_as(D)


@pytest.fixture(scope="module")
def libs():
    ref = pyoracle.ref_primitives()
    orc = pyoracle.oracle_primitives()
    for L, pre in ((ref, "ref_"), (orc, "orc_")):
        getattr(L, pre + "tone_map").restype = C.c_double
        getattr(L, pre + "tone_map").argtypes = [C.c_double, C.c_double]
        getattr(L, pre + "tone_map_derivative").restype = C.c_double
        getattr(L, pre + "tone_map_derivative").argtypes = [C.c_double, C.c_double]
    return ref, orc


def test_rng_streams(libs):
    ref, orc = libs
    for keys in ([], [7], [3, 0x9E01], [1, 0x9E02, 12345]):
        k = (C.c_uint64 * max(1, len(keys)))(*keys)
        a = (C.c_uint64 * 8)()
        b = (C.c_uint64 * 8)()
        ref.ref_rng(C.c_uint64(42), len(keys), k, 8, a)
        orc.orc_rng(C.c_uint64(42), len(keys), k, 8, b)
        assert list(a) == list(b)
    # the package's numpy RNG (used for synthetic inputs) is the same stream
    r = S.Rng(42, 3, 0x9E01)
    a = (C.c_uint64 * 2)()
    ref.ref_rng(C.c_uint64(42), 2, (C.c_uint64 * 2)(3, 0x9E01), 2, a)
    assert int(r.next_u64()) == a[0] and int(r.next_u64()) == a[1]


def test_pixel_positions_and_rays(libs):
    ref, orc = libs
    cam = S.sample_views_on_sphere(3, 2.5, 11, 40.0, 37, 23)[1]
    cc = cdr_camera(tuple(cam.origin), tuple(cam.right), tuple(cam.up), tuple(cam.forward), cam.fov_deg,
                    cam.width, cam.height)
    a = (C.c_double * 3)()
    b = (C.c_double * 3)()
    for spp in (1, 4, 5, 9, 16):
        for (px, py, s) in ((0, 0, 0), (5, 7, spp - 1), (36, 22, spp // 2)):
            ref.ref_pixel_sample_position(C.c_uint64(9), 3, px, py, 37, s, spp, a)
            orc.orc_pixel_sample_position(C.c_uint64(9), 3, px, py, 37, s, spp, b)
            assert list(a)[:2] == list(b)[:2]
            ref.ref_primary_ray(C.byref(cc), C.c_double(a[0]), C.c_double(a[1]), a)
            orc.orc_primary_ray(C.byref(cc), C.c_double(b[0]), C.c_double(b[1]), b)
            assert list(a) == list(b)
    rng = np.random.default_rng(0)
    for _ in range(50):
        p = rng.normal(size=3)
        qa, qb = (C.c_double * 2)(), (C.c_double * 2)()
        da, db = C.c_double(), C.c_double()
        ra = ref.ref_project(C.byref(cc), dp(p), qa, C.byref(da))
        rb = orc.orc_project(C.byref(cc), dp(p), qb, C.byref(db))
        assert ra == rb and da.value == db.value
        if ra:
            assert list(qa) == list(qb)
        ja, jb = (C.c_double * 6)(), (C.c_double * 6)()
        ref.ref_projection_jacobian(C.byref(cc), dp(p), ja)
        orc.orc_projection_jacobian(C.byref(cc), dp(p), jb)
        assert list(ja) == list(jb)


def test_brdf_texture_tonemap(libs):
    ref, orc = libs
    rng = np.random.default_rng(2)
    oa, ob = (C.c_double * 11)(), (C.c_double * 11)()
    for _ in range(300):
        ad, as_ = rng.uniform(0, 1, 3), rng.uniform(0, 0.3, 3)
        alpha, mu = rng.uniform(0.01, 1), rng.uniform(-0.2, 1)
        ref.ref_eval_brdf(dp(ad), dp(as_), C.c_double(alpha), C.c_double(mu), oa)
        orc.orc_eval_brdf(dp(ad), dp(as_), C.c_double(alpha), C.c_double(mu), ob)
        assert list(oa) == list(ob)
    tex = rng.uniform(0, 1, size=(6, 5, 3)).astype(np.float32).astype(np.float64)
    ta, tb = (C.c_double * 13)(), (C.c_double * 13)()
    ia, ib = (C.c_int32 * 4)(), (C.c_int32 * 4)()
    for ch, data in ((3, tex), (1, tex[..., 0].copy())):
        for _ in range(200):
            u, v = rng.uniform(-2, 3, 2)
            ref.ref_sample_texture(dp(data), 5, 6, ch, C.c_double(u), C.c_double(v), ta, ia)
            orc.orc_sample_texture(dp(data), 5, 6, ch, C.c_double(u), C.c_double(v), tb, ib)
            assert list(ta) == list(tb) and list(ia) == list(ib)
    for v in (-0.5, 0.0, 1e-9, 0.3, 0.5, 0.999, 1.0, 2.5):
        for g in (1.0, 2.2):
            assert ref.ref_tone_map(v, g) == orc.orc_tone_map(v, g)
            assert ref.ref_tone_map_derivative(v, g) == orc.orc_tone_map_derivative(v, g)


def test_ray_triangle_shared(libs):
    ref, orc = libs
    rng = np.random.default_rng(3)
    a, b = (C.c_double * 3)(), (C.c_double * 3)()
    for _ in range(500):
        o, d = rng.normal(size=3), rng.normal(size=3)
        d /= np.linalg.norm(d)
        p0, p1, p2 = rng.normal(size=(3, 3))
        ha = ref.ref_ray_triangle(dp(o), dp(d), dp(p0), dp(p1), dp(p2), a)
        hb = orc.orc_ray_triangle(dp(o), dp(d), dp(p0), dp(p1), dp(p2), b)
        assert ha == hb
        if ha:
            assert list(a) == list(b)


@pytest.fixture(scope="module")
def scene():
    return small_scene(freq=5, tex=16, views=2, image=32)


def test_views_and_edges_match_reference(scene):
    r = RefLib(scene)
    np.testing.assert_array_equal(r.edges(), scene.mesh.edges)   # build_adjacency order
    cams = np.zeros(4, dtype=pyoracle.cdr_camera * 1)
    out = (cdr_camera * 4)()
    r.lib.ref_sample_views_on_sphere(4, C.c_double(2.5), C.c_uint64(11), C.c_double(40.0), 64, 48, out)
    mine = S.sample_views_on_sphere(4, 2.5, 11, 40.0, 64, 48)
    for k in range(4):
        for f in ("origin", "right", "up", "forward"):
            np.testing.assert_allclose(list(getattr(out[k], f)), getattr(mine[k], f), rtol=0, atol=1e-15)
    del cams


def test_normals_tmin_intersections(scene):
    o, r = Oracle(scene), RefLib(scene)
    np.testing.assert_array_equal(o.vertex_normals(), r.vertex_normals())
    assert o.t_min == r.t_min
    rng = np.random.default_rng(4)
    orig = rng.normal(size=(2000, 3)) * 1.5
    dirs = -orig + rng.normal(size=(2000, 3)) * 0.3
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    a = o.intersect(orig, dirs)
    b = o.intersect(orig, dirs, brute=True)
    c = r.intersect(orig, dirs)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)
    np.testing.assert_array_equal(a[0], c[0])
    hit = a[0] >= 0
    for x, y in zip(a[1:], c[1:]):
        np.testing.assert_array_equal(x[hit], y[hit])


@pytest.mark.parametrize("spp", [1, 4, 9])
def test_render_loss_interior_boundary(scene, spp):
    o, r = Oracle(scene), RefLib(scene)
    seed = 5
    tg = targets_for(scene, spp, seed, Oracle)
    lay = layout_for(scene, optimize_light=True)
    for v in range(2):
        ao, mo, ho = o.render(v, spp, seed)
        ar, mr, hr = r.render(v, spp, seed)
        np.testing.assert_array_equal(ho, hr)
        np.testing.assert_array_equal(mo, mr)
        np.testing.assert_array_equal(ao, ar)
        lo, adjo = o.view_loss(ao, tg[v])
        lr, adjr = r.view_loss(ar, tg[v])
        assert lo == lr
        np.testing.assert_array_equal(adjo, adjr)
        np.testing.assert_array_equal(o.interior(v, adjo, spp, seed, ho, lay), r.interior(v, adjr, spp, seed, hr, lay))
        so, to = o.silhouettes(v)
        sr, tr = r.silhouettes(v)
        assert to == tr and len(so) == len(sr)
        for k in so.dtype.names:
            np.testing.assert_array_equal(so[k], sr[k])
        for probe in (0, 1):
            go, do = o.boundary(v, adjo, 32 * 32, seed, lay, probe=probe)
            gr, dr = r.boundary(v, adjr, 32 * 32, seed, lay, probe=probe)
            assert do == dr
            np.testing.assert_array_equal(go, gr)


def test_laplacian_both_modes(scene):
    o, r = Oracle(scene), RefLib(scene)
    for mode in (0, 1):
        vo, go, mo = o.laplacian(mode, 0.37)
        vr, gr, mr = r.laplacian(mode, 0.37)
        assert vo == vr
        np.testing.assert_array_equal(go, gr)
        for x, y in zip(mo, mr):
            np.testing.assert_array_equal(x, y)


def test_total_loss_hot_subset():
    sc = blob_scene(freq=6, tex=16, views=2, image=32)
    o, r = Oracle(sc), RefLib(sc)
    spp, seed = 4, 3
    tg = targets_for(sc, spp, seed, Oracle)
    lay = layout_for(sc)
    lo, go, ro = o.loss_grad(tg, settings(spp, seed), lay, want_rendered=True)
    bd, gr, rr = r.total_loss(tg, spp, seed, lay, want_rendered=True)
    assert lo[0] == bd[1] and lo[1] == bd[2]
    np.testing.assert_array_equal(go, gr)
    np.testing.assert_array_equal(ro, rr)


def test_icosphere_generator_matches_reference():
    """scenes.icosphere restates make_icosphere (mesh.cpp:270-298) exactly."""
    import ctypes as C2
    L = pyoracle.ref_primitives()
    for sub in (0, 1, 2, 3):
        nv, nt = C2.c_int32(), C2.c_int32()
        L.ref_make_mesh(0, sub, C2.c_double(0.5), C2.c_uint64(0), C2.byref(nv), C2.byref(nt), None, None, None)
        pos = np.zeros((nv.value, 3))
        uv = np.zeros((nv.value, 2))
        tris = np.zeros((nt.value, 3), np.int32)
        L.ref_make_mesh(0, sub, C2.c_double(0.5), C2.c_uint64(0), C2.byref(nv), C2.byref(nt), dp(pos),
                        uv.ctypes.data_as(D), tris.ctypes.data_as(C2.POINTER(C2.c_int32)))
        m = S.icosphere(sub, 0.5)
        np.testing.assert_array_equal(m.triangles, tris)
        np.testing.assert_allclose(m.positions, pos, rtol=0, atol=1e-15)
