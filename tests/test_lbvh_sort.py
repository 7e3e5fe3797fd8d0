"""The LBVH's hand-written radix sort (prepare.cu k_sort_hist / k_sort_pass):
the leaf keys must equal a full sort of the Morton|face keys, computed here
with the same fp64 arithmetic as k_bbox_* / k_morton (so every key is known
exactly), on meshes of one to ~50 tiles, with heavy Morton ties (stability),
after positions change (per-iteration rebuild)."""
import numpy as np
import pytest

from paper_2103_15208_b200 import scenes as S
from paper_2103_15208_b200.api import Renderer

pytestmark = pytest.mark.gpu


def _expand(v):
    v = v.astype(np.uint64)
    v = (v * np.uint64(0x00010001)) & np.uint64(0xFF0000FF)
    v = (v * np.uint64(0x00000101)) & np.uint64(0x0F00F00F)
    v = (v * np.uint64(0x00000011)) & np.uint64(0xC30C30C3)
    v = (v * np.uint64(0x00000005)) & np.uint64(0x49249249)
    return v


def expected_keys(pos, tris):
    lo, hi = pos.min(axis=0), pos.max(axis=0)
    p = pos[tris]  # T x 3 x 3
    cen = 0.5 * (p.min(axis=1) + p.max(axis=1))
    ext = hi - lo
    q = []
    for k in range(3):
        u = (cen[:, k] - lo[k]) / ext[k] if ext[k] > 0 else np.full(len(tris), 0.5)
        qi = np.trunc(u * 1024.0).astype(np.int64)
        q.append(np.clip(qi, 0, 1023))
    m = (_expand(q[0]) << np.uint64(2)) | (_expand(q[1]) << np.uint64(1)) | _expand(q[2])
    keys = (m << np.uint64(32)) | np.arange(len(tris), dtype=np.uint64)
    return np.sort(keys)


def _mesh_scene(mesh):
    d, s, r = S.random_maps(8)
    return S.Scene(mesh, d, s, r, S.sample_views_on_sphere(1, 2.5, 11, 40, 16, 16))


@pytest.mark.parametrize("make", [lambda: S.geodesic_sphere(1), lambda: S.geodesic_sphere(4), lambda: S.blob(16),
                                  lambda: S.blob(59), lambda: S.torus_knot()])
def test_lbvh_keys_are_the_full_sort(make):
    m = make()
    r = Renderer(0, _mesh_scene(m))
    got = r.lbvh_keys()
    np.testing.assert_array_equal(got, expected_keys(m.positions, m.triangles))
    # per-iteration rebuild after the positions move
    rng = np.random.default_rng(3)
    pos2 = m.positions + rng.normal(scale=1e-3, size=m.positions.shape)
    r.update_positions(pos2)
    np.testing.assert_array_equal(r.lbvh_keys(), expected_keys(pos2, m.triangles))


def test_lbvh_sort_is_stable_under_ties():
    """Many triangles with one centroid cell: equal Morton codes must keep
    ascending face order across tile boundaries (3 tiles of 4,096 keys)."""
    n = 10000
    rng = np.random.default_rng(5)
    pos = np.concatenate([rng.uniform(0.4999, 0.5001, size=(3 * n, 3)), [[0, 0, 0], [1, 1, 1], [1, 0, 1]]])
    tris = np.arange(3 * n, dtype=np.int32).reshape(n, 3)
    tris = np.concatenate([tris, [[3 * n, 3 * n + 1, 3 * n + 2]]]).astype(np.int32)
    m = S.Mesh(pos, tris, None)
    r = Renderer(0, _mesh_scene(m))
    got = r.lbvh_keys()
    exp = expected_keys(pos, tris)
    np.testing.assert_array_equal(got, exp)
    assert len(np.unique(exp >> np.uint64(32))) < n // 4  # the case really has ties
