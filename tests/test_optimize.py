"""Resident optimiser: adam_step (adam.cpp:9-54) + apply
(params.cpp:103-134) and robust_evolve (evolve.cpp:19-53) on the device.

Pins: reference (oracle/_ref) -> tests/golden/optimize.npz -> oracle (C) ->
GPU. All of it is bit-exact: element-wise fp64 in the reference's operation
order, bias corrections with the host's pow, exact self-intersection answers.
"""
import os

import numpy as np
import pytest

from oracle.pyoracle import adam_step, layout_for, robust_evolve
from paper_2103_15208_b200 import scenes as S

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "optimize.npz")
EVOLVE_CASES = 7


def _z():
    return np.load(GOLD)


def _adam_scene():
    return S.make_scene(S.icosphere(2), 8, 1, 16)


# ---------------------------------------------------------------- oracle (CPU)
@pytest.mark.parametrize("light", (0, 1))
@pytest.mark.parametrize("step", (0, 6))
def test_oracle_adam_matches_golden(light, step):
    z = _z()
    sc = _adam_scene()
    lay = layout_for(sc, optimize_light=bool(light))
    k = f"adam_l{light}_s{step}"
    rc, st, m2, v2, p2, d2 = adam_step(z["adam_cfg"], lay, sc.mesh.V, (8, 8), step, z[f"{k}_m"], z[f"{k}_v"],
                                       z[f"{k}_params"], z[f"{k}_grad"])
    assert rc == 0 and st == int(z[f"{k}_step2"])
    for a, b in ((m2, "m2"), (v2, "v2"), (p2, "p2"), (d2, "d2")):
        np.testing.assert_array_equal(a, z[f"{k}_{b}"])


def test_oracle_adam_rejects_nonfinite():
    sc = _adam_scene()
    lay = layout_for(sc)
    n = lay["total"]
    g = np.zeros(n)
    g[5] = np.nan
    rc = adam_step((0.9, 0.999, 1e-8, 1e-3, 1e-2, 1e-2), lay, sc.mesh.V, (8, 8), 0, np.zeros(n), np.zeros(n),
                   np.zeros(n), g)[0]
    assert rc == 2  # CDR_ERR_NONFINITE (adam.cpp:12-13)


@pytest.mark.parametrize("case", range(EVOLVE_CASES))
def test_oracle_evolve_matches_golden(case):
    z = _z()
    rc, pos, scale = robust_evolve(z["evolve_pos"], z["evolve_tris"], z[f"evolve{case}_d"])
    assert rc == int(z[f"evolve{case}_rc"]) and scale == float(z[f"evolve{case}_scale"])
    np.testing.assert_array_equal(pos, z[f"evolve{case}_pos"])


def test_oracle_evolve_rejects_self_intersecting_input():
    z = _z()
    rc = robust_evolve(z["evolve_bad_pos"], z["evolve_bad_tris"], np.zeros_like(z["evolve_bad_pos"]))[0]
    assert rc == int(z["evolve_bad_rc"]) == 7


@pytest.mark.ref
def test_oracle_adam_and_evolve_match_reference_random():
    rng = np.random.default_rng(31)
    sc = _adam_scene()
    for light in (False, True):
        lay = layout_for(sc, optimize_light=light)
        n = lay["total"]
        args = (rng.normal(0, 0.1, n), rng.uniform(0, 0.1, n), rng.uniform(-0.1, 1.1, n), rng.normal(0, 3, n))
        cfg = (0.8, 0.99, 1e-6, 5e-3, 3e-2, 1e-1)
        a = adam_step(cfg, lay, sc.mesh.V, (8, 8), 2, *args)
        b = adam_step(cfg, lay, sc.mesh.V, (8, 8), 2, *args, ref=True)
        assert a[:2] == b[:2]
        for x, y in zip(a[2:], b[2:]):
            np.testing.assert_array_equal(x, y)
    m = S.geodesic_sphere(6)
    for sd in (0.01, 0.1, 1.0):
        d = rng.normal(0, sd, m.positions.shape)
        a, b = robust_evolve(m.positions, m.triangles, d), robust_evolve(m.positions, m.triangles, d, ref=True)
        assert a[0] == b[0] and a[2] == b[2]
        np.testing.assert_array_equal(a[1], b[1])


# ---------------------------------------------------------------- GPU
def _targets(sc, spp, seed):
    from paper_2103_15208_b200.api import RenderSettings, Renderer
    tr = Renderer(0, S.perturbed_target_scene(sc))
    out = [tr.render(k, RenderSettings(spp=spp, seed=seed + 0x7A9), want_hits=False)[0] for k in range(len(sc.cameras))]
    tr.close()
    return out


def _pack(sc, lay):
    p = np.zeros(lay["total"])
    V = sc.mesh.V
    p[lay["positions"]:lay["positions"] + 3 * V] = sc.mesh.positions.ravel()
    n = sc.diffuse.shape[0] * sc.diffuse.shape[1]
    p[lay["diffuse"]:lay["diffuse"] + 3 * n] = sc.diffuse.ravel()
    p[lay["specular"]:lay["specular"] + 3 * n] = sc.specular.ravel()
    p[lay["roughness"]:lay["roughness"] + n] = sc.roughness.ravel()
    if lay["light"] >= 0:
        p[lay["light"]:lay["light"] + 3] = sc.light
    return p


@pytest.mark.gpu
@pytest.mark.parametrize("light", (False, True))
def test_gpu_resident_loop_matches_oracle(light):
    """total_loss -> adam_step -> evolve, three iterations, entirely on the
    device; every step checked bit for bit against the oracle fed the same
    device gradient."""
    from paper_2103_15208_b200.api import AdamConfig, RenderSettings, Renderer
    sc = S.make_scene(S.blob(4), 16, 2, 32)
    spp, seed = 4, 3
    tg = _targets(sc, spp, seed)
    r = Renderer(0, sc)
    for k, t in enumerate(tg):
        r.set_target(k, t)
    lay = layout_for(sc, optimize_light=light)
    cfg = AdamConfig(lr_positions=2e-3, lr_textures=5e-2, lr_light=0.5)
    r.adam_init(cfg, lay)
    params = _pack(sc, lay)
    n = lay["total"]
    m, v, step = np.zeros(n), np.zeros(n), 0
    st = RenderSettings(spp=spp, seed=seed)
    views = np.arange(len(sc.cameras))
    tris = sc.mesh.triangles
    for it in range(3):
        r.loss_grad(views, st, lay, device_only=True)
        g = r.get_grad(n)
        disp, gstep = r.adam_step()
        rc, step, m, v, params, d2 = adam_step(cfg.tuple(), lay, sc.mesh.V, sc.tex_res, step, m, v, params, g)
        assert rc == 0 and gstep == step
        np.testing.assert_array_equal(disp, d2)
        gm, gv, _ = r.adam_state()
        np.testing.assert_array_equal(gm, m)
        np.testing.assert_array_equal(gv, v)
        scale, gpos = r.evolve()
        P = lay["positions"]
        pos = params[P:P + 3 * sc.mesh.V].reshape(-1, 3)
        rc, opos, oscale = robust_evolve(pos, tris, d2)
        assert rc == 0 and scale == oscale
        np.testing.assert_array_equal(gpos, opos)
        params[P:P + 3 * sc.mesh.V] = opos.ravel()
        np.testing.assert_array_equal(r.params(lay), params)
    # the resident state is what the next pass renders: equal to a fresh
    # renderer built from the packed parameters (bit-exact images)
    n_tex = sc.diffuse.shape[0] * sc.diffuse.shape[1]
    th, tw = sc.diffuse.shape[:2]
    fresh = S.Scene(S.Mesh(params[P:P + 3 * sc.mesh.V].reshape(-1, 3), tris, sc.mesh.uvs, sc.mesh.edges),
                    params[lay["diffuse"]:lay["diffuse"] + 3 * n_tex].reshape(th, tw, 3),
                    params[lay["specular"]:lay["specular"] + 3 * n_tex].reshape(th, tw, 3),
                    params[lay["roughness"]:lay["roughness"] + n_tex].reshape(th, tw), sc.cameras,
                    params[lay["light"]:lay["light"] + 3] if light else sc.light, sc.background)
    r2 = Renderer(0, fresh)
    for k in range(len(sc.cameras)):
        a = r.render(k, st)
        b = r2.render(k, st)
        np.testing.assert_array_equal(a[0], b[0])
        np.testing.assert_array_equal(a[2], b[2])


@pytest.mark.gpu
def test_gpu_adam_matches_golden():
    from paper_2103_15208_b200.api import AdamConfig
    z = _z()
    sc = _adam_scene()
    cfg = AdamConfig(*z["adam_cfg"])
    for light in (0, 1):
        lay = layout_for(sc, optimize_light=bool(light))
        for step in (0, 6):
            k = f"adam_l{light}_s{step}"
            r = _renderer_with_params(sc, lay, z[f"{k}_params"])
            r.adam_init(cfg, lay)
            r.set_adam_state(z[f"{k}_m"], z[f"{k}_v"], step)
            r.set_grad(z[f"{k}_grad"])
            disp, st = r.adam_step()
            assert st == int(z[f"{k}_step2"])
            np.testing.assert_array_equal(disp, z[f"{k}_d2"])
            m, v, _ = r.adam_state()
            np.testing.assert_array_equal(m, z[f"{k}_m2"])
            np.testing.assert_array_equal(v, z[f"{k}_v2"])
            p = r.params(lay)
            P = lay["positions"]
            want = z[f"{k}_p2"].copy()
            np.testing.assert_array_equal(p[P + 3 * sc.mesh.V:], want[P + 3 * sc.mesh.V:])


def _renderer_with_params(sc, lay, params):
    from paper_2103_15208_b200.api import Renderer
    n = sc.diffuse.shape[0] * sc.diffuse.shape[1]
    th, tw = sc.diffuse.shape[:2]
    P = lay["positions"]
    s2 = S.Scene(sc.mesh, params[lay["diffuse"]:lay["diffuse"] + 3 * n].reshape(th, tw, 3),
                 params[lay["specular"]:lay["specular"] + 3 * n].reshape(th, tw, 3),
                 params[lay["roughness"]:lay["roughness"] + n].reshape(th, tw), sc.cameras,
                 params[lay["light"]:lay["light"] + 3] if lay["light"] >= 0 else sc.light, sc.background)
    del P
    return Renderer(0, s2)


@pytest.mark.gpu
@pytest.mark.parametrize("case", range(EVOLVE_CASES))
def test_gpu_evolve_matches_golden(case):
    from paper_2103_15208_b200.api import Renderer
    z = _z()
    m = S.Mesh(z["evolve_pos"], z["evolve_tris"], np.zeros((len(z["evolve_pos"]), 2)))
    d, s, rr = S.constant_maps(4, (0.5, 0.5, 0.5), (0.05, 0.05, 0.05), 0.5)
    r = Renderer(0, S.Scene(m, d, s, rr, S.sample_views_on_sphere(1, 2.5, 11, 40, 8, 8)))
    scale, pos = r.evolve(z[f"evolve{case}_d"])
    assert scale == float(z[f"evolve{case}_scale"])
    np.testing.assert_array_equal(pos, z[f"evolve{case}_pos"])


@pytest.mark.gpu
def test_gpu_evolve_rejects_self_intersecting_input():
    from paper_2103_15208_b200.api import InputSelfIntersecting, Renderer
    z = _z()
    m = S.Mesh(z["evolve_bad_pos"], z["evolve_bad_tris"], np.zeros((len(z["evolve_bad_pos"]), 2)))
    d, s, rr = S.constant_maps(4, (0.5, 0.5, 0.5), (0.05, 0.05, 0.05), 0.5)
    r = Renderer(0, S.Scene(m, d, s, rr, S.sample_views_on_sphere(1, 2.5, 11, 40, 8, 8)))
    with pytest.raises(InputSelfIntersecting):
        r.evolve(np.zeros_like(z["evolve_bad_pos"]))


@pytest.mark.gpu
def test_gpu_optimiser_and_query_errors():
    """Error behaviour of the new entry points, as the reference's exceptions."""
    from paper_2103_15208_b200.api import AdamConfig, CollodiffError, NonFiniteGradient, Renderer, SizeMismatch
    sc = _adam_scene()
    r = Renderer(0, sc)
    lay = layout_for(sc)
    with pytest.raises(CollodiffError):  # no optimiser state yet
        r.adam_step()
    r.adam_init(AdamConfig(), lay)
    with pytest.raises(SizeMismatch):  # no gradient of this layout yet (adam.cpp:10-11)
        r.adam_step()
    g = np.zeros(lay["total"])
    g[3] = np.inf
    r.set_grad(g)
    before = r.params(lay)
    with pytest.raises(NonFiniteGradient):  # adam.cpp:12-13: nothing is updated
        r.adam_step()
    np.testing.assert_array_equal(r.params(lay), before)
    m, v, step = r.adam_state()
    assert step == 0 and not m.any() and not v.any()
    bad = sc.mesh.triangles.copy()
    bad[0, 0] = sc.mesh.V + 5
    with pytest.raises(CollodiffError):
        r.self_intersects(sc.mesh.positions, bad)
    with pytest.raises(CollodiffError):
        r.closest_points(sc.mesh.positions, bad, np.zeros((1, 3)))
