"""GPU parity: libcdr.so (through the C-ABI) against the CPU oracle on identical
inputs and the shared counter-RNG stream.

Bars (BASELINE.json north_star): triangle-ID and visibility buffers bit-exact;
images within 1e-5 relative L2; vertex and texel gradients within 1e-4
relative L2. Silhouette segment sets are required bit-exact too (the boundary
pass's importance sampling depends on them).
"""
import numpy as np
import pytest

from oracle.pyoracle import Oracle, RefLib, SEGMENT_DTYPE as ORC_SEG
from paper_2103_15208_b200 import scenes as S
from paper_2103_15208_b200.api import (NonFiniteGradient, RenderSettings, Renderer, SizeMismatch,
                                       param_layout)
from tests.scenes_util import blob_scene, rel_l2, small_scene, targets_for

pytestmark = pytest.mark.gpu

IMG_TOL = 1e-5
GRAD_TOL = 1e-4   # the contract (north star)
GRAD_TIGHT = 1e-9  # fused-path assertions: only fp64 RED order differs (measured ~1e-15)


def _pair(scene):
    return Renderer(0, scene), Oracle(scene)


def _seg_equal(a, b):
    assert len(a) == len(b)
    for k in ORC_SEG.names:
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)


@pytest.fixture(scope="module")
def sphere():
    return small_scene(freq=5, tex=16, views=3, image=40)


def test_normals_and_tmin_bit_exact(sphere):
    r, o = _pair(sphere)
    np.testing.assert_array_equal(r.vertex_normals(), o.vertex_normals())


@pytest.mark.parametrize("spp", [1, 4, 9, 16])
def test_render_bit_exact(sphere, spp):
    r, o = _pair(sphere)
    st = RenderSettings(spp=spp, seed=3)
    for v in range(len(sphere.cameras)):
        rg, mg, hg = r.render(v, st)
        ro, mo, ho = o.render(v, spp, 3)
        np.testing.assert_array_equal(hg, ho)      # triangle IDs: bit-exact
        np.testing.assert_array_equal(mg, mo)      # visibility mask: bit-exact
        assert rel_l2(rg, ro) <= IMG_TOL
        # fp32-representable textures + unfused fp64: the image is bit-exact too
        np.testing.assert_array_equal(rg, ro)


def test_radiance_at_matches(sphere):
    r, o = _pair(sphere)
    rng = np.random.default_rng(0)
    xy = rng.uniform(0, 40, size=(500, 2))
    a, ta = r.radiance_at(1, xy)
    b, tb = o.radiance_at(1, xy)
    np.testing.assert_array_equal(ta, tb)
    assert rel_l2(a, b) <= IMG_TOL


def test_view_loss(sphere):
    r, o = _pair(sphere)
    rng = np.random.default_rng(1)
    a = rng.uniform(-0.1, 1.2, size=(40, 40, 3))
    t = rng.uniform(0, 1, size=(40, 40, 3))
    m = (rng.uniform(size=(40, 40)) > 0.3).astype(np.float64)
    for mask, use in ((None, False), (m, True)):
        vg, ag = r.view_rendering_loss(a, t, 0.7, 2.2, mask, use)
        vo, ao = o.view_loss(a, t, mask, 0.7, 2.2, use)
        assert abs(vg - vo) <= 1e-12 * abs(vo)
        assert rel_l2(ag, ao) <= 1e-12
    v0, a0 = r.view_rendering_loss(a, t, 0.0)
    assert v0 == 0 and not a0.any()
    with pytest.raises(SizeMismatch):
        r.view_rendering_loss(a, t[:20])


@pytest.mark.parametrize("light", [False, True])
def test_interior_pass(sphere, light):
    r, o = _pair(sphere)
    spp, seed = 4, 5
    tg = targets_for(sphere, spp, seed, Oracle)
    lay = param_layout(sphere, optimize_light=light)
    for v in range(len(sphere.cameras)):
        img, _, hit = o.render(v, spp, seed)
        _, adj = o.view_loss(img, tg[v])
        go = o.interior(v, adj, spp, seed, hit, lay)
        gg = r.interior_pass(v, adj, RenderSettings(spp=spp, seed=seed), hit, lay)
        ntex = sphere.tex_res[0] * sphere.tex_res[1]
        sizes = {"positions": 3 * sphere.mesh.V, "diffuse": 3 * ntex, "specular": 3 * ntex, "roughness": ntex}
        for name, n in sizes.items():
            a0 = lay[name]
            assert rel_l2(gg[a0:a0 + n], go[a0:a0 + n]) <= GRAD_TOL, name
            assert rel_l2(gg[a0:a0 + n], go[a0:a0 + n]) <= GRAD_TIGHT, name
        if light:
            assert rel_l2(gg[-3:], go[-3:]) <= GRAD_TIGHT
    with pytest.raises(SizeMismatch):
        r.interior_pass(0, adj, RenderSettings(spp=spp, seed=seed), hit[:-1], lay)


def test_silhouettes_bit_exact(sphere):
    r, o = _pair(sphere)
    for v in range(len(sphere.cameras)):
        sg, tg = r.extract_silhouettes(v)
        so, to = o.silhouettes(v)
        _seg_equal(sg, so)
        assert tg == to


@pytest.mark.parametrize("probe", [0, 1])
def test_boundary_pass(sphere, probe):
    r, o = _pair(sphere)
    spp, seed = 4, 9
    tg = targets_for(sphere, spp, seed, Oracle)
    lay = param_layout(sphere)
    for v in range(len(sphere.cameras)):
        img, _, _ = o.render(v, spp, seed)
        _, adj = o.view_loss(img, tg[v])
        go, do = o.boundary(v, adj, 40 * 40, seed, lay, probe=probe)
        gg, dg = r.boundary_pass(v, adj, 40 * 40, seed, lay, probe=probe)
        assert dg == do
        assert np.linalg.norm(go) > 0
        assert rel_l2(gg, go) <= GRAD_TOL
        # the draws are the reference's exactly (same CDF, same lower_bound):
        # only the order of the fp64 deposits differs
        assert rel_l2(gg, go) <= 1e-9


def _loss_grad_check(scene, spp, seed, lay, use_mask=False, masks=None, lam_lap=0.1, bterm=True, bsamples=0):
    r, o = _pair(scene)
    tg = targets_for(scene, spp, seed, Oracle)
    st = RenderSettings(spp=spp, seed=seed, boundary_term=bterm, boundary_samples=bsamples)
    from oracle.pyoracle import settings as osettings
    lo, go, ro = o.loss_grad(tg, osettings(spp, seed, boundary_term=int(bterm), boundary_samples=bsamples), lay,
                             lam_lap=lam_lap, targets_mask=masks, use_mask=use_mask, want_rendered=True)
    for k in range(len(scene.cameras)):
        r.set_target(k, tg[k], None if masks is None else masks[k])
    lg, gg, stats, rg = r.loss_grad(np.arange(len(scene.cameras)), st, lay, 1.0, lam_lap, 0, use_mask,
                                    want_rendered=True)
    np.testing.assert_array_equal(rg, ro.ravel())
    assert abs(lg[0] - lo[0]) <= 1e-10 * max(1e-300, abs(lo[0]))
    assert abs(lg[1] - lo[1]) <= 1e-10 * max(1e-300, abs(lo[1]))
    pos = slice(lay["positions"], lay["positions"] + 3 * scene.mesh.V)
    tex = slice(lay["diffuse"], lay["total"])
    assert rel_l2(gg[pos], go[pos]) <= GRAD_TOL
    assert rel_l2(gg[tex], go[tex]) <= GRAD_TOL
    assert rel_l2(gg[pos], go[pos]) <= GRAD_TIGHT, rel_l2(gg[pos], go[pos])
    assert rel_l2(gg[tex], go[tex]) <= GRAD_TIGHT, rel_l2(gg[tex], go[tex])
    assert stats.samples == sum(c.width * c.height for c in scene.cameras) * spp
    return stats


def test_loss_grad_matches_oracle(sphere):
    st = _loss_grad_check(sphere, 4, 1, param_layout(sphere))
    assert st.hit_samples > 0 and st.adjoint_samples > 0 and st.boundary_active > 0


def test_loss_grad_blob_selfoccluding():
    sc = blob_scene(freq=8, tex=32, views=2, image=48)
    _loss_grad_check(sc, 4, 2, param_layout(sc, optimize_light=True))


def test_loss_grad_spp16_background_empty_tiles():
    # spp 16: beam tiles with no candidate take k_render's background path
    # (no hit-cache traffic); a non-zero background exercises its mean and tone
    # map, 46 x 46 images leave partial edge tiles, masks the masked loss
    sc = small_scene(freq=5, tex=16, views=2, image=46)
    sc.background = np.array([0.1, 0.2, 0.3])
    rng = np.random.default_rng(5)
    masks = (rng.uniform(size=(2, 46, 46)) > 0.2).astype(np.float64)
    st = _loss_grad_check(sc, 16, 3, param_layout(sc), use_mask=True, masks=masks)
    assert 0 < st.shaded_samples < st.samples  # the background path ran
    st = _loss_grad_check(sc, 16, 5, param_layout(sc))
    assert 0 < st.shaded_samples < st.samples


def test_loss_grad_masks_and_options(sphere):
    rng = np.random.default_rng(3)
    masks = (rng.uniform(size=(3, 40, 40)) > 0.2).astype(np.float64)
    _loss_grad_check(sphere, 4, 1, param_layout(sphere), use_mask=True, masks=masks)
    _loss_grad_check(sphere, 1, 4, param_layout(sphere), lam_lap=0.0, bterm=False)
    _loss_grad_check(sphere, 9, 4, param_layout(sphere), bsamples=333)


def test_laplacian(sphere):
    r, o = _pair(sphere)
    for mode in (0, 1):
        vo, go, (oo, io, xo) = o.laplacian(mode, 0.3)
        og, ig, xg = r.cotangent_laplacian(mode)
        np.testing.assert_array_equal(og, oo)
        np.testing.assert_array_equal(ig, io)
        np.testing.assert_array_equal(xg, xo)
        vg, gg = r.laplacian_loss(mode, 0.3)
        assert abs(vg - vo) <= 1e-12 * abs(vo)
        np.testing.assert_array_equal(gg, go)


def test_empty_scene_renders_background():
    # render.cpp / test_render.cpp:67-76: no triangles -> zero image and mask
    m = S.Mesh(np.zeros((0, 3)), np.zeros((0, 3), np.int32), np.zeros((0, 2)))
    d, s, rr = S.constant_maps(4, (1, 1, 1), (0, 0, 0), 0.5)
    sc = S.Scene(m, d, s, rr, S.sample_views_on_sphere(1, 2.5, 11, 40, 16, 16))
    r = Renderer(0, sc)
    img, mask, hit = r.render(0, RenderSettings(spp=4))
    assert not img.any() and not mask.any() and (hit == -1).all()


def test_mixed_view_sizes_and_global_ids():
    sc = small_scene(freq=4, tex=8, views=2, image=24)
    sc.cameras[1] = S.look_at(sc.cameras[1].origin, [0, 0, 0], [0, 0, 1], 35.0, 31, 17)
    ids = [5, 2]
    r = Renderer(0, sc, view_ids=ids)
    o = Oracle(sc, view_ids=ids)
    for v in range(2):
        a = r.render(v, RenderSettings(spp=4, seed=8))
        b = o.render(v, 4, 8)
        np.testing.assert_array_equal(a[2], b[2])
        np.testing.assert_array_equal(a[0], b[0])


def test_nonfinite_gradient_is_reported():
    sc = small_scene(freq=3, tex=8, views=1, image=16)
    sc.light = np.array([np.inf, 1.0, 1.0])
    r = Renderer(0, sc)
    o = Oracle(sc)
    img, _, hit = o.render(0, 4, 1)
    adj = np.full((16, 16, 3), 1e-3)
    with pytest.raises(NonFiniteGradient):
        r.interior_pass(0, adj, RenderSettings(spp=4, seed=1), hit, param_layout(sc))


@pytest.mark.ref
def test_gpu_matches_reference_directly(sphere):
    """Straight against the reference compiled from its own sources."""
    ref = RefLib(sphere)
    r = Renderer(0, sphere)
    spp, seed = 4, 1
    lay = param_layout(sphere)
    tg = targets_for(sphere, spp, seed, Oracle)
    bd, gr, rr = ref.total_loss(tg, spp, seed, lay, want_rendered=True)
    bd_g, gg, rend = r.total_loss(list(tg), RenderSettings(spp=spp, seed=seed), lay)
    assert abs(bd_g["rend"] - bd[1]) <= 1e-10 * bd[1]
    assert abs(bd_g["lap"] - bd[2]) <= 1e-10 * bd[2]
    pos = slice(0, 3 * sphere.mesh.V)
    assert rel_l2(gg[pos], gr[pos]) <= GRAD_TOL
    assert rel_l2(gg[pos.stop:], gr[pos.stop:]) <= GRAD_TOL
    assert rel_l2(gg[pos], gr[pos]) <= GRAD_TIGHT
    assert rel_l2(gg[pos.stop:], gr[pos.stop:]) <= GRAD_TIGHT
    for v in range(len(sphere.cameras)):
        np.testing.assert_array_equal(r.render(v, RenderSettings(spp=spp, seed=seed))[2],
                                      ref.render(v, spp, seed)[2])


def test_grazing_rays_near_silhouettes_exact(sphere):
    """Rays within a few ulps to 1e-3 px of silhouette edges (the boundary
    probes' regime, where BVH pruning and the fp32 pre-test are most
    stressed): triangle IDs must equal the exact oracle's."""
    sc = blob_scene(freq=8, tex=16, views=2, image=64)
    r, o = _pair(sc)
    rng = np.random.default_rng(7)
    for v in range(2):
        segs, _ = o.silhouettes(v)
        t = rng.uniform(0, 1, size=(len(segs), 8))
        q0, q1 = segs["q0"][:, None, :], segs["q1"][:, None, :]
        pts = q0 + (q1 - q0) * t[..., None]
        tang = (q1 - q0) / np.linalg.norm(q1 - q0, axis=-1, keepdims=True)
        nrm = np.stack([-tang[..., 1], tang[..., 0]], axis=-1)
        offs = rng.choice([0.0, 1e-12, -1e-12, 1e-9, -1e-9, 1e-6, -1e-6, 1e-3, -1e-3, 0.5, -0.5],
                          size=t.shape)[..., None]
        xy = (pts + nrm * offs).reshape(-1, 2)
        _, tg = r.radiance_at(v, xy)
        _, to = o.radiance_at(v, xy)
        np.testing.assert_array_equal(tg, to)


def test_grad_overwrite_flag(sphere):
    """CDR_FLAG_GRAD_OVERWRITE writes the fresh gradient; the default adds."""
    r, _ = _pair(sphere)
    spp, seed = 4, 1
    tg = targets_for(sphere, spp, seed, Oracle)
    for k in range(len(sphere.cameras)):
        r.set_target(k, tg[k])
    lay = param_layout(sphere)
    views = np.arange(len(sphere.cameras))
    st = RenderSettings(spp=spp, seed=seed)
    _, g0, _, _ = r.loss_grad(views, st, lay)
    junk = np.full(lay["total"], 7.0)
    _, g1, _, _ = r.loss_grad(views, st, lay, grad=junk.copy(), overwrite=True)
    assert rel_l2(g1, g0) <= 1e-12  # runs differ only by fp64 RED order
    _, g2, _, _ = r.loss_grad(views, st, lay, grad=junk.copy())
    assert rel_l2(g2 - 7.0, g0) <= 1e-12


def test_get_rendered_matches_pass_outputs(sphere):
    """cdr_get_rendered returns the images the last loss pass rendered."""
    r, _ = _pair(sphere)
    spp, seed = 4, 2
    tg = targets_for(sphere, spp, seed, Oracle)
    for k in range(len(sphere.cameras)):
        r.set_target(k, tg[k])
    lay = param_layout(sphere)
    _, _, _, rend = r.loss_grad(np.arange(len(sphere.cameras)), RenderSettings(spp=spp, seed=seed), lay,
                                want_rendered=True)
    off = 0
    for v, cam in enumerate(sphere.cameras):
        n = cam.width * cam.height * 3
        rgb, mask = r.rendered(v)
        np.testing.assert_array_equal(rgb.ravel(), rend[off:off + n])
        img, m2, _ = r.render(v, RenderSettings(spp=spp, seed=seed))
        np.testing.assert_array_equal(mask, m2)
        off += n


def test_fp32_targets_equal_widened_fp64(sphere):
    """cdr_set_target_f32 (PFM data) == cdr_set_target of the widened doubles."""
    spp, seed = 4, 6
    tg = targets_for(sphere, spp, seed, Oracle)
    rng = np.random.default_rng(2)
    lay = param_layout(sphere)
    views = np.arange(len(sphere.cameras))
    st = RenderSettings(spp=spp, seed=seed)
    t32 = [t.astype(np.float32) for t in tg]
    m32 = [(rng.uniform(size=t.shape[:2]) > 0.3).astype(np.float32) * np.float32(0.75) for t in tg]
    out = []
    for f32 in (False, True):
        r, _ = _pair(sphere)
        for k in range(len(sphere.cameras)):
            if f32:
                r.set_target(k, t32[k], m32[k])
            else:
                r.set_target(k, t32[k].astype(np.float64), m32[k].astype(np.float64))
        loss, g, _, _ = r.loss_grad(views, st, lay, use_target_mask=True)
        out.append((loss, g))
    # the per-view loss is an fp64 RED sum across CTAs: equal to rounding
    np.testing.assert_allclose(out[0][0], out[1][0], rtol=1e-12, atol=0)
    assert rel_l2(out[0][1], out[1][1]) <= 1e-12


@pytest.mark.parametrize("fast_cap,big_cap,split_cap", [("0", None, None), ("3", None, None), ("3", "8", None),
                                                         ("0", "0", None), ("2", "4", "1"), ("0", "0", "0")])
def test_big_tile_lists_exact(sphere, monkeypatch, fast_cap, big_cap, split_cap):
    """Tiles over the fast pass's candidate cap are rebuilt by the big pass
    (255 candidates, 128-entry pixel lists); tiles over that are split into
    quadrant lists (k_tile_lists_split). Forcing (almost) every tile through
    those passes must leave hit caches and images bit-exact and gradients in
    tolerance."""
    monkeypatch.setenv("CDR_BEAM_FAST_CAP", fast_cap)
    if big_cap is not None:
        monkeypatch.setenv("CDR_BEAM_BIG_CAP", big_cap)
    if split_cap is not None:  # quadrants overflow too: split once more, then the huge pass
        monkeypatch.setenv("CDR_BEAM_SPLIT_CAP", split_cap)
    blob = blob_scene(freq=8, tex=32, views=2, image=48)
    for sc in (sphere, blob):
        r, o = _pair(sc)
        for spp in (4, 16):
            st = RenderSettings(spp=spp, seed=5)
            for v in range(len(sc.cameras)):
                rgb, mask, hit = r.render(v, st)
                ro, mo, ho = o.render(v, spp, 5)
                np.testing.assert_array_equal(hit, ho)
                np.testing.assert_array_equal(mask, mo)
                np.testing.assert_array_equal(rgb, ro)
    # (with every tile forced into it, the big queue, sized for 1/16 of the
    # tiles, overflows too: those tiles are traced per ray, also exact)
    _loss_grad_check(sphere, 16, 2, param_layout(sphere))


@pytest.mark.parametrize("fast_cap", [None, "3"])
def test_block_queue_lists_exact(monkeypatch, fast_cap):
    """The list builder over k_top_walk's queue of non-empty 2 x 2 tile blocks
    (the empty blocks' tiles written by k_top_walk itself), with and without
    tiles forced through the big pass: hit caches, images, the loss call and
    the probes through its lists exact."""
    monkeypatch.setenv("CDR_BLOCK_QUEUE", "1")
    if fast_cap is not None:
        monkeypatch.setenv("CDR_BEAM_FAST_CAP", fast_cap)
    sc = blob_scene(freq=8, tex=16, views=2, image=64)
    r, o = _pair(sc)
    for spp in (4, 16):
        st = RenderSettings(spp=spp, seed=8)
        for v in range(len(sc.cameras)):
            rgb, mask, hit = r.render(v, st)
            ro, mo, ho = o.render(v, spp, 8)
            np.testing.assert_array_equal(hit, ho)
            np.testing.assert_array_equal(rgb, ro)
    _loss_grad_check(sc, 16, 8, param_layout(sc))
    tg = targets_for(sc, 16, 8, Oracle)
    for k in range(len(sc.cameras)):
        r.set_target(k, tg[k])
    r.loss_grad(np.arange(len(sc.cameras)), RenderSettings(spp=16, seed=8), param_layout(sc))
    rng = np.random.default_rng(17)
    for v in range(len(sc.cameras)):
        xy = _silhouette_probe_points(o, v, rng)
        cg, tgp = r.probe_points(v, xy)
        co, to = o.radiance_at(v, xy)
        np.testing.assert_array_equal(tgp, to)
        np.testing.assert_array_equal(cg, co)


@pytest.mark.parametrize("wh", [(37, 29), (29, 37)])
def test_odd_image_sizes_exact(wh):
    """Partial tiles at the right and bottom edges, odd tile counts (the 2x2
    tile blocks of the list builder, the 4x2-pixel shading CTAs, the half-tile
    trace CTAs): hit caches and images bit-exact, gradients in tolerance."""
    w, h = wh
    m = S.blob(6)
    d, s_, r_ = S.random_maps(16)
    sc = S.Scene(m, d, s_, r_, S.sample_views_on_sphere(2, 2.5, 11, 40, w, h))
    r, o = _pair(sc)
    for spp in (16, 4):
        st = RenderSettings(spp=spp, seed=9)
        for v in range(len(sc.cameras)):
            rgb, mask, hit = r.render(v, st)
            ro, mo, ho = o.render(v, spp, 9)
            np.testing.assert_array_equal(hit, ho)
            np.testing.assert_array_equal(mask, mo)
            np.testing.assert_array_equal(rgb, ro)
    _loss_grad_check(sc, 16, 3, param_layout(sc))


@pytest.mark.parametrize("knob", ["CDR_NO_BEAM", "CDR_CHUNK_MB", "CDR_NO_SHARED_TOP", "CDR_NO_SPLIT", "CDR_NO_QUEUE",
                                  "CDR_NO_HUGE", "CDR_NO_TOP_PREPASS",
                                  "CDR_TRACE_QUEUE", "CDR_NO_TRACE_QUEUE", "CDR_BLOCK_QUEUE", "CDR_NO_BLOCK_QUEUE"])
def test_alternate_paths_exact(sphere, monkeypatch, knob):
    """The A/B switches kept in the code (per-ray traversal only; view chunks
    through lists -> trace -> shade; every tile from the BVH root) stay exact."""
    monkeypatch.setenv(knob, "1")
    blob = blob_scene(freq=8, tex=32, views=2, image=48)
    r, o = _pair(blob)
    st = RenderSettings(spp=16, seed=4)
    for v in range(len(blob.cameras)):
        rgb, mask, hit = r.render(v, st)
        ro, mo, ho = o.render(v, 16, 4)
        np.testing.assert_array_equal(hit, ho)
        np.testing.assert_array_equal(rgb, ro)
    _loss_grad_check(blob, 16, 4, param_layout(blob))


def _silhouette_probe_points(o, v, rng, per_seg=8):
    """Continuous points around every silhouette segment of view v at normal
    offsets +/-{0, 1e-12, 1e-9, 1e-6, 1e-3, 0.5} px, interleaved as the
    boundary pass's probe pairs (x - n/2, x + n/2) plus raw offsets."""
    segs, _ = o.silhouettes(v)
    t = rng.uniform(0, 1, size=(len(segs), per_seg))
    q0, q1 = segs["q0"][:, None, :], segs["q1"][:, None, :]
    pts = q0 + (q1 - q0) * t[..., None]
    tang = (q1 - q0) / np.linalg.norm(q1 - q0, axis=-1, keepdims=True)
    nrm = np.stack([-tang[..., 1], tang[..., 0]], axis=-1)
    offs = rng.choice([0.0, 1e-12, -1e-12, 1e-9, -1e-9, 1e-6, -1e-6, 1e-3, -1e-3, 0.5, -0.5],
                      size=t.shape)[..., None]
    raw = (pts + nrm * offs).reshape(-1, 2)
    pairs = np.stack([pts - 0.5 * nrm, pts + 0.5 * nrm], axis=-2).reshape(-1, 2)  # k_boundary's xm, xp
    return np.concatenate([pairs, raw, raw[:1]])  # odd count: the last point goes alone


@pytest.mark.parametrize("spp", [4, 16])
@pytest.mark.parametrize("fast_cap", [None, "0", "split", "split2"])
def test_probe_points_through_lists_bit_exact(monkeypatch, spp, fast_cap):
    """The boundary probes of the fused loss call trace through the per-pixel
    candidate lists (trace_points2, beam.cuh), not per-ray traversal. After a
    loss call, points at +/-{0 .. 0.5} px around every silhouette, traced by
    that same path, must hit exactly the oracle's triangles and return its
    radiance. fast_cap "0" sends every tile through the big-list pass (and its
    overflow to per-ray traversal)."""
    if fast_cap == "split":  # every tile through the big pass, most of them split into quadrants
        monkeypatch.setenv("CDR_BEAM_FAST_CAP", "0")
        monkeypatch.setenv("CDR_BEAM_BIG_CAP", "6")
    elif fast_cap == "split2":  # and most quadrants split once more
        monkeypatch.setenv("CDR_BEAM_FAST_CAP", "0")
        monkeypatch.setenv("CDR_BEAM_BIG_CAP", "6")
        monkeypatch.setenv("CDR_BEAM_SPLIT_CAP", "2")
    elif fast_cap is not None:
        monkeypatch.setenv("CDR_BEAM_FAST_CAP", fast_cap)
    sc = blob_scene(freq=8, tex=16, views=2, image=64)
    r, o = _pair(sc)
    tg = targets_for(sc, spp, 3, Oracle)
    for k in range(len(sc.cameras)):
        r.set_target(k, tg[k])
    r.loss_grad(np.arange(len(sc.cameras)), RenderSettings(spp=spp, seed=3), param_layout(sc))
    rng = np.random.default_rng(11)
    for v in range(len(sc.cameras)):
        xy = _silhouette_probe_points(o, v, rng)
        cg, tgp = r.probe_points(v, xy)
        co, to = o.radiance_at(v, xy)
        np.testing.assert_array_equal(tgp, to)
        np.testing.assert_array_equal(cg, co)
        assert (to >= 0).any() and (to < 0).any()


def test_probe_points_needs_lists(sphere):
    r, _ = _pair(sphere)
    from paper_2103_15208_b200.api import CollodiffError
    with pytest.raises(CollodiffError):
        r.probe_points(0, np.zeros((2, 2)))


def test_context_memory_is_returned():
    """cdr_destroy frees every device buffer (DBuf owns its allocation)."""
    import torch
    sc = blob_scene(freq=8, tex=64, views=2, image=96)
    tg = targets_for(sc, 16, 1, Oracle)

    def cycle():
        r = Renderer(0, sc)
        for k in range(2):
            r.set_target(k, tg[k])
        lay = param_layout(sc)
        r.loss_grad([0, 1], RenderSettings(spp=16, seed=1), lay)
        r.regularisers(__import__("paper_2103_15208_b200.api", fromlist=["LossWeights"]).LossWeights(), lay)
        r.self_intersects(sc.mesh.positions, sc.mesh.triangles)
        r.close()

    cycle()  # first use: CUDA context, module load
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info(0)[0]
    for _ in range(3):
        cycle()
    torch.cuda.synchronize()
    free1 = torch.cuda.mem_get_info(0)[0]
    assert free0 - free1 < 8 << 20, (free0 - free1)


def test_rejected_mesh_keeps_previous_state(sphere):
    """cdr_set_mesh validates everything before it changes the context."""
    from paper_2103_15208_b200.api import _dp, _ip
    r, o = _pair(sphere)
    st = RenderSettings(spp=4, seed=2)
    h0 = r.render(0, st)[2]
    pos = np.ascontiguousarray(sphere.mesh.positions[:10])
    nonmanifold = np.array([[0, 1, 2], [0, 1, 3], [0, 1, 4]], np.int32)  # edge (0, 1) in three faces
    assert r.L.cdr_set_mesh(r.h, _dp(pos), len(pos), _ip(nonmanifold), 3, None, None, 0) != 0
    assert "non-manifold" in r.L.cdr_last_error(r.h).decode()
    P = np.ascontiguousarray(sphere.mesh.positions)
    T = np.ascontiguousarray(sphere.mesh.triangles, dtype=np.int32)
    bad_edges = np.array([[0, 1, 0, 10 ** 6]], np.int32)  # a caller edge whose face is out of range
    assert r.L.cdr_set_mesh(r.h, _dp(P), len(P), _ip(T), len(T), None, _ip(bad_edges), 1) != 0
    assert "face out of range" in r.L.cdr_last_error(r.h).decode()
    np.testing.assert_array_equal(r.render(0, st)[2], h0)
    np.testing.assert_array_equal(h0, o.render(0, 4, 2)[2])


def test_boundary_pass_caller_segments_larger_than_edges(sphere):
    """A caller-supplied silhouette set with more segments than the mesh has
    edges (segments repeated) is sized and strided by max(E, nseg); segment
    vertices out of range are rejected."""
    from paper_2103_15208_b200.api import CollodiffError
    r, o = _pair(sphere)
    spp, seed = 4, 9
    tg = targets_for(sphere, spp, seed, Oracle)
    lay = param_layout(sphere)
    img, _, _ = o.render(0, spp, seed)
    _, adj = o.view_loss(img, tg[0])
    segs, _ = o.silhouettes(0)
    E = len(r.edges())
    reps = E // len(segs) + 2
    big = np.concatenate([segs] * reps)
    assert len(big) > E
    gg, _ = r.boundary_pass(0, adj, 40 * 40, seed, lay, segments=big)
    go, _ = o.boundary(0, adj, 40 * 40, seed, lay, segments=big)
    assert rel_l2(gg, go) <= GRAD_TIGHT
    bad = segs.copy()
    bad["v1"][0] = 10 ** 7
    with pytest.raises(CollodiffError):
        r.boundary_pass(0, adj, 40 * 40, seed, lay, segments=bad)
