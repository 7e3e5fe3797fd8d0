"""cdr_stage_params: the loss call reads the staged positions and maps itself
(maps uploaded on the copy stream beside the visibility pass; with pinned
buffers the map/light gradient and the images come down beside the boundary
pass). The results must be bit-identical to cdr_update_positions +
cdr_set_textures before the call with the gradient downloaded at its end —
for pinned and pageable buffers, the canonical layout and a permuted one
(positions last, light in the middle), and total_loss with the regularisers
(whose map gradient is added before the early download)."""
import ctypes as C

import numpy as np
import pytest

from paper_2103_15208_b200 import api
from paper_2103_15208_b200 import scenes as S
from paper_2103_15208_b200.api import LossWeights, RenderSettings, Renderer

pytestmark = pytest.mark.gpu


def _pinned(shape):
    import torch
    return torch.zeros(shape, dtype=torch.float64).pin_memory().numpy()


def _scene():
    return S.make_scene(S.blob(3), 64, 3, 64)


def _renderer(scene, light=False):
    r = Renderer(0, scene)
    tr = Renderer(0, S.perturbed_target_scene(scene))
    for k in range(len(scene.cameras)):
        r.set_target(k, tr.render(k, RenderSettings(spp=4, seed=77), want_hits=False)[0])
    tr.close()
    return r


def _permuted_layout(scene):
    """positions last, light between the maps (a valid, non-canonical ParamLayout)"""
    n = scene.tex_res[0] * scene.tex_res[1]
    lay, off = {}, 0
    for name, size in (("diffuse", 3 * n), ("light", 3), ("specular", 3 * n), ("roughness", n),
                       ("positions", 3 * scene.mesh.V)):
        lay[name] = off
        off += size
    lay["total"] = off
    return lay


def _params(scene, step):
    rng = np.random.default_rng(step)
    pos = scene.mesh.positions + 1e-3 * rng.standard_normal(scene.mesh.positions.shape)
    d = np.clip(scene.diffuse + 0.05 * rng.standard_normal(scene.diffuse.shape), 0, 1)
    s = np.clip(scene.specular + 0.05 * rng.standard_normal(scene.specular.shape), 0, 1)
    ro = np.clip(scene.roughness + 0.05 * rng.standard_normal(scene.roughness.shape), 0.05, 1)
    return pos, d, s, ro


def _total_loss(r, views, st, lay, w, grad, rend):
    s = st.c()
    s.flags |= api.CDR_FLAG_GRAD_OVERWRITE
    bd = np.zeros(7)
    reg = w.c_reg()
    lc = api._clayout(lay)
    r._chk(r.L.cdr_total_loss(r.h, api._ip(views), len(views), C.byref(s), w.rend, w.lap, C.byref(reg), 0, 0,
                              C.byref(lc), api._dp(bd), api._dp(grad), api._dp(rend), None, None))
    return bd


@pytest.mark.parametrize("pinned", [True, False])
@pytest.mark.parametrize("permuted", [False, True])
def test_staged_loss_grad_identical(pinned, permuted):
    sc = _scene()
    lay = _permuted_layout(sc) if permuted else api.param_layout(sc, optimize_light=True)
    views = np.arange(len(sc.cameras), dtype=np.int32)
    st = RenderSettings(spp=4, seed=5)
    npx = sum(c.width * c.height for c in sc.cameras)
    a, b = _renderer(sc), _renderer(sc)
    for step in range(3):  # the staged maps change every step, as under Adam
        pos, d, s, ro = _params(sc, step)
        a.update_positions(pos)
        a.set_textures(d, s, ro)
        la, ga, _, ra = a.loss_grad(views, st, lay, overwrite=True, want_rendered=True)
        g = _pinned(lay["total"]) if pinned else np.zeros(lay["total"])
        rend = _pinned(3 * npx) if pinned else np.zeros(3 * npx)
        g[:] = np.nan  # overwrite: every entry is written
        if pinned:
            pp, dp, sp, rp = _pinned(pos.shape), _pinned(d.shape), _pinned(s.shape), _pinned(ro.shape)
            pp[:], dp[:], sp[:], rp[:] = pos, d, s, ro
            pos, d, s, ro = pp, dp, sp, rp
        b.stage_params(pos, (d, s, ro))
        lb, gb, _, rb = b.loss_grad(views, st, lay, grad=g, overwrite=True, rendered_out=rend)
        # the per-view loss sums are fp64 atomics (order varies run to run)
        np.testing.assert_allclose(lb, la, rtol=1e-13)
        np.testing.assert_array_equal(ra, rb)
        # fp64 atomics: the same deposits in a different order may differ in the last bits
        np.testing.assert_allclose(gb, ga, rtol=1e-12, atol=1e-300)
    a.close()
    b.close()


def test_staged_total_loss_with_regularisers():
    sc = _scene()
    lay = api.param_layout(sc)
    views = np.arange(len(sc.cameras), dtype=np.int32)
    st = RenderSettings(spp=4, seed=9)
    w = LossWeights()
    npx = sum(c.width * c.height for c in sc.cameras)
    a, b = _renderer(sc), _renderer(sc)
    pos, d, s, ro = _params(sc, 11)
    a.update_positions(pos)
    a.set_textures(d, s, ro)
    ga, rda = np.zeros(lay["total"]), np.zeros(3 * npx)
    bda = _total_loss(a, views, st, lay, w, ga, rda)
    pp, dp, sp, rp = _pinned(pos.shape), _pinned(d.shape), _pinned(s.shape), _pinned(ro.shape)
    pp[:], dp[:], sp[:], rp[:] = pos, d, s, ro
    gb, rdb = _pinned(lay["total"]), _pinned(3 * npx)
    b.stage_params(pp, (dp, sp, rp))
    bdb = _total_loss(b, views, st, lay, w, gb, rdb)
    np.testing.assert_allclose(bdb, bda, rtol=1e-13)
    np.testing.assert_array_equal(rda, rdb)
    np.testing.assert_allclose(gb, ga, rtol=1e-12, atol=1e-300)
    nt = sc.tex_res[0] * sc.tex_res[1]
    assert np.any(gb[lay["specular"]:lay["specular"] + 3 * nt] != 0)  # the regularisers' map terms are in
    a.close()
    b.close()


def test_staged_params_applied_by_other_entry_points():
    """A render after cdr_stage_params sees the staged parameters."""
    sc = _scene()
    a, b = _renderer(sc), _renderer(sc)
    pos, d, s, ro = _params(sc, 3)
    a.update_positions(pos)
    a.set_textures(d, s, ro)
    b.stage_params(pos, (d, s, ro))
    st = RenderSettings(spp=4, seed=1)
    np.testing.assert_array_equal(a.render(0, st)[0], b.render(0, st)[0])
    a.close()
    b.close()


def test_staged_params_cleared_on_error():
    sc = _scene()
    r = _renderer(sc)
    lay = api.param_layout(sc)
    base = r.render(0, RenderSettings(spp=4, seed=1))[0]
    pos, d, s, ro = _params(sc, 4)
    r.stage_params(pos, (d, s, ro))
    with pytest.raises(Exception):
        r.loss_grad(np.array([99], dtype=np.int32), RenderSettings(spp=4, seed=1), lay)
    # the failed call consumed nothing: the next call renders the old parameters
    np.testing.assert_array_equal(r.render(0, RenderSettings(spp=4, seed=1))[0], base)
    # maps are all or none (C-ABI: CDR_ERR_INVALID_ARG; the Python mirror raises first)
    dd = np.ascontiguousarray(d)
    assert r.L.cdr_stage_params(r.h, None, api._dp(dd), None, api._dp(dd), 64, 64) == 5
    with pytest.raises(ValueError):
        r.stage_params(None, (d, None, ro))
    r.close()


@pytest.mark.parametrize("nviews", [1, 3, 5])
def test_grouped_shading_image_downloads(nviews):
    """Queue-mode loss calls (spp 16) with page-locked image destinations
    shade in up to 16 view groups and download each group's images and
    masks while the next group shades: the same images, masks, loss and
    gradient as with pageable destinations (downloaded after the call)."""
    sc = S.make_scene(S.blob(3), 32, nviews, 48)
    lay = api.param_layout(sc)
    views = np.arange(nviews, dtype=np.int32)
    st = RenderSettings(spp=16, seed=7)
    npx = sum(c.width * c.height for c in sc.cameras)
    a, b = _renderer(sc), _renderer(sc)
    for _ in range(2):  # the second call runs with the sizes of the first (queue mode either way)
        rga, mka = np.zeros(3 * npx), np.zeros(npx)
        la, ga, _, _ = a.loss_grad(views, st, lay, overwrite=True, rendered_out=rga, mask_out=mka)
        rgb, mkb, gb = _pinned(3 * npx), _pinned(npx), _pinned(lay["total"])
        rgb[:] = np.nan
        mkb[:] = np.nan
        lb, _, _, _ = b.loss_grad(views, st, lay, grad=gb, overwrite=True, rendered_out=rgb, mask_out=mkb)
        np.testing.assert_array_equal(rgb, rga)
        np.testing.assert_array_equal(mkb, mka)
        np.testing.assert_allclose(lb, la, rtol=1e-13)
        np.testing.assert_allclose(gb, ga, rtol=1e-12, atol=1e-300)
    a.close()
    b.close()
