"""Images stay bit-exact for maps off the fp32 grid.

Shading reads fp32 texel records when every map value is fp32-representable
(the fast path) and fp64 records otherwise (k_pack_textures flags the maps;
the shading kernels are compiled for both). Maps after optimiser steps are
off the grid: these tests perturb the synthetic maps by ~1e-9 and require the
renders, the loss call's images, the probe radiance through the candidate
lists and the gradients to match the oracle (fp64 maps) as before — images
bit for bit — and the fp32 path to come back once the maps are on the grid
again."""
import dataclasses

import numpy as np
import pytest

from oracle.pyoracle import Oracle, settings as osettings
from paper_2103_15208_b200.api import RenderSettings, Renderer, param_layout
from tests.scenes_util import blob_scene, rel_l2, targets_for

pytestmark = pytest.mark.gpu

GRAD_TIGHT = 1e-9


def _off_grid(scene, seed=5):
    rng = np.random.default_rng(seed)
    jig = lambda m: np.clip(m + 1e-9 * rng.standard_normal(m.shape), 1e-3, 1.0)
    sc = dataclasses.replace(scene, diffuse=jig(scene.diffuse), specular=jig(scene.specular),
                             roughness=jig(scene.roughness))
    assert np.any(sc.diffuse.astype(np.float32).astype(np.float64) != sc.diffuse)
    return sc


@pytest.fixture(scope="module")
def blob():
    return _off_grid(blob_scene(freq=8, tex=16, views=2, image=48))


@pytest.mark.parametrize("spp", [1, 16])
def test_render_off_grid_maps_bit_exact(blob, spp):
    r, o = Renderer(0, blob), Oracle(blob)
    st = RenderSettings(spp=spp, seed=3)
    for v in range(len(blob.cameras)):
        rg, mg, hg = r.render(v, st)
        ro, mo, ho = o.render(v, spp, 3)
        np.testing.assert_array_equal(hg, ho)
        np.testing.assert_array_equal(rg, ro)
    xy = np.random.default_rng(1).uniform(0, 48, size=(257, 2))
    cg, tg = r.radiance_at(0, xy)
    co, to = o.radiance_at(0, xy)
    np.testing.assert_array_equal(tg, to)
    np.testing.assert_array_equal(cg, co)
    r.close()


@pytest.mark.parametrize("spp", [4, 16])
def test_loss_grad_off_grid_maps(blob, spp):
    r, o = Renderer(0, blob), Oracle(blob)
    lay = param_layout(blob)
    tg = targets_for(blob, spp, 2, Oracle)
    lo, go, ro = o.loss_grad(tg, osettings(spp, 2), lay, want_rendered=True)
    for k in range(len(blob.cameras)):
        r.set_target(k, tg[k])
    lg, gg, _, rg = r.loss_grad(np.arange(len(blob.cameras)), RenderSettings(spp=spp, seed=2), lay,
                                want_rendered=True)
    np.testing.assert_array_equal(rg, ro.ravel())  # the loss call's images, bit for bit
    assert abs(lg[0] - lo[0]) <= 1e-12 * abs(lo[0])
    P = 3 * blob.mesh.V
    assert rel_l2(gg[:P], go[:P]) <= GRAD_TIGHT
    assert rel_l2(gg[P:], go[P:]) <= GRAD_TIGHT
    # the probe radiance through the candidate lists of that call
    xy = np.random.default_rng(4).uniform(0, 48, size=(301, 2))
    cg, tgp = r.probe_points(0, xy)
    co, to = o.radiance_at(0, xy)
    np.testing.assert_array_equal(tgp, to)
    np.testing.assert_array_equal(cg, co)
    r.close()


def test_switches_back_to_fp32_records():
    """On-grid maps again -> the fp32 records (same image as a fresh context)."""
    base = blob_scene(freq=8, tex=16, views=1, image=48)
    off = _off_grid(base)
    r = Renderer(0, off)
    st = RenderSettings(spp=4, seed=1)
    img_off = r.render(0, st)[0]
    np.testing.assert_array_equal(img_off, Oracle(off).render(0, 4, 1)[0])
    r.set_textures(base.diffuse, base.specular, base.roughness)
    img = r.render(0, st)[0]
    fresh = Renderer(0, base)
    np.testing.assert_array_equal(img, fresh.render(0, st)[0])
    np.testing.assert_array_equal(img, Oracle(base).render(0, 4, 1)[0])
    assert np.any(img != img_off)
    r.close()
    fresh.close()


def test_adam_step_moves_maps_off_grid_and_stays_exact():
    """After a resident Adam step the maps are off the fp32 grid; the render
    of the updated maps equals the oracle's render of the same maps."""
    from paper_2103_15208_b200.api import AdamConfig
    sc = blob_scene(freq=8, tex=16, views=2, image=48)
    r = Renderer(0, sc)
    lay = param_layout(sc)
    tg = targets_for(sc, 4, 2, Oracle)
    for k in range(len(sc.cameras)):
        r.set_target(k, tg[k])
    r.adam_init(AdamConfig(lr_positions=0.0), lay)
    r.loss_grad(np.arange(len(sc.cameras)), RenderSettings(spp=4, seed=2), lay, device_only=True)
    r.adam_step(want_displacement=False)
    params = r.params(lay)
    n = sc.diffuse.size // 3
    d = params[lay["diffuse"]:lay["diffuse"] + 3 * n].reshape(sc.diffuse.shape)
    s = params[lay["specular"]:lay["specular"] + 3 * n].reshape(sc.specular.shape)
    ro = params[lay["roughness"]:lay["roughness"] + n].reshape(sc.roughness.shape)
    assert np.any(d.astype(np.float32).astype(np.float64) != d)
    moved = dataclasses.replace(sc, diffuse=d, specular=s, roughness=ro)
    img = r.render(0, RenderSettings(spp=4, seed=9))[0]
    np.testing.assert_array_equal(img, Oracle(moved).render(0, 4, 9)[0])
    r.close()
