"""Fixtures produced by the reference library itself (tests/golden/make_golden.py
on oracle/_ref). They travel with the repo, so the oracle and the GPU path are
pinned to the reference even where /root/reference is absent."""
import glob
import os

import numpy as np
import pytest

from oracle.pyoracle import Oracle, layout_for
from paper_2103_15208_b200 import scenes as S

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
# scene fixtures (selfint.npz / optimize.npz: tests/test_selfint.py, tests/test_optimize.py)
FIXTURES = sorted(f for f in glob.glob(os.path.join(HERE, "*.npz")) if os.path.basename(f) not in ("selfint.npz", "optimize.npz", "closest.npz"))


def load(path):
    z = np.load(path)
    m = S.Mesh(z["positions"], z["triangles"], z["uvs"], z["edges"])
    cams = []
    for c in z["cameras"]:
        cams.append(S.Camera(np.array(c["origin"]), np.array(c["right"]), np.array(c["up"]),
                             np.array(c["forward"]), float(c["fov_deg"]), int(c["width"]), int(c["height"])))
    sc = S.Scene(m, z["diffuse"], z["specular"], z["roughness"], cams, z["light"], z["background"])
    return z, sc


def rel_l2(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(np.asarray(a) - b) / (nb if nb > 0 else 1.0)


@pytest.mark.parametrize("path", FIXTURES, ids=os.path.basename)
def test_oracle_reproduces_reference_fixture(path):
    z, sc = load(path)
    o = Oracle(sc)
    spp, seed = int(z["spp"]), int(z["seed"])
    lay = layout_for(sc, optimize_light=bool(z["optimize_light"]))
    for v in range(len(sc.cameras)):
        rgb, mask, hit = o.render(v, spp, seed)
        np.testing.assert_array_equal(hit, z[f"v{v}_hit"])
        np.testing.assert_array_equal(mask, z[f"v{v}_mask"])
        np.testing.assert_array_equal(rgb, z[f"v{v}_rgb"])
        val, adj = o.view_loss(rgb, z["targets"][v])
        assert val == float(z[f"v{v}_loss"])
        np.testing.assert_array_equal(adj, z[f"v{v}_adj"])
        np.testing.assert_array_equal(o.interior(v, adj, spp, seed, hit, lay), z[f"v{v}_interior"])
        segs, tot = o.silhouettes(v)
        assert tot == float(z[f"v{v}_seglen"])
        for k in segs.dtype.names:
            np.testing.assert_array_equal(segs[k], z[f"v{v}_segments"][k])
        g, deg = o.boundary(v, adj, sc.cameras[v].width * sc.cameras[v].height, seed, lay)
        np.testing.assert_array_equal(g, z[f"v{v}_boundary"])
        assert deg == int(z[f"v{v}_degenerate"])
    val, grad, (oo, ii, xx) = o.laplacian(0, 0.1)
    assert val == float(z["lap_value"])
    np.testing.assert_array_equal(grad, z["lap_grad"])
    np.testing.assert_array_equal(xx, z["lap_vals"])


@pytest.mark.gpu
@pytest.mark.parametrize("path", FIXTURES, ids=os.path.basename)
def test_gpu_reproduces_reference_fixture(path):
    from paper_2103_15208_b200.api import RenderSettings, Renderer
    z, sc = load(path)
    r = Renderer(0, sc)
    spp, seed = int(z["spp"]), int(z["seed"])
    lay = layout_for(sc, optimize_light=bool(z["optimize_light"]))
    st = RenderSettings(spp=spp, seed=seed)
    for v in range(len(sc.cameras)):
        rgb, mask, hit = r.render(v, st)
        np.testing.assert_array_equal(hit, z[f"v{v}_hit"])      # bit-exact
        np.testing.assert_array_equal(mask, z[f"v{v}_mask"])    # bit-exact
        assert rel_l2(rgb, z[f"v{v}_rgb"]) <= 1e-5
        segs, tot = r.extract_silhouettes(v)
        for k in segs.dtype.names:
            np.testing.assert_array_equal(segs[k], z[f"v{v}_segments"][k])
        adj = z[f"v{v}_adj"]
        assert rel_l2(r.interior_pass(v, adj, st, hit, lay), z[f"v{v}_interior"]) <= 1e-4
        g, _ = r.boundary_pass(v, adj, sc.cameras[v].width * sc.cameras[v].height, seed, lay)
        assert rel_l2(g, z[f"v{v}_boundary"]) <= 1e-4
    bd, g, _ = r.total_loss(list(z["targets"]), st, lay)
    assert abs(bd["rend"] - z["total_breakdown"][1]) <= 1e-10 * z["total_breakdown"][1]
    assert abs(bd["lap"] - z["total_breakdown"][2]) <= 1e-10 * z["total_breakdown"][2]
    P = 3 * sc.mesh.V
    assert rel_l2(g[:P], z["total_grad"][:P]) <= 1e-4
    assert rel_l2(g[P:], z["total_grad"][P:]) <= 1e-4
