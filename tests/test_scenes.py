"""Synthetic-input generators: the named shapes and their invariants."""
import numpy as np
import pytest

from paper_2103_15208_b200 import scenes as S
from paper_2103_15208_b200.shard import laplacian_weight, shard_views, weak_views


@pytest.mark.parametrize("freq,V,T,E", [(11, 1212, 2420, 3630), (59, 34812, 69620, 104430)])
def test_geodesic_counts(freq, V, T, E):
    m = S.geodesic_sphere(freq) if freq < 59 else S.blob(freq)
    assert (m.V, m.T, m.E) == (V, T, E)
    assert (m.edges[:, 3] >= 0).all()  # closed 2-manifold


def test_outward_orientation_and_uvs():
    for m in (S.geodesic_sphere(11), S.blob(16)):
        P, F = m.positions, m.triangles
        n = np.cross(P[F[:, 1]] - P[F[:, 0]], P[F[:, 2]] - P[F[:, 0]])
        assert ((n * P[F].mean(axis=1)).sum(axis=1) > 0).mean() > 0.99
        assert (m.uvs >= 0).all() and (m.uvs <= 1).all()


def test_torus_knot():
    k = S.torus_knot(200, 20)
    assert (k.V, k.T, k.E) == (4000, 8000, 12000)
    assert (k.edges[:, 3] >= 0).all()
    assert np.abs(k.positions).max() <= 0.6


def test_edges_sorted_like_std_map():
    m = S.geodesic_sphere(5)
    keys = m.edges[:, 0].astype(np.int64) * m.V + m.edges[:, 1]
    assert (np.diff(keys) > 0).all() and (m.edges[:, 0] < m.edges[:, 1]).all()
    assert (m.edges[:, 2] < np.where(m.edges[:, 3] < 0, np.inf, m.edges[:, 3])).all()


def test_textures_are_fp32_exact_and_in_range():
    d, s, r = S.random_maps(64)
    for a, lo, hi in ((d, 0.2, 0.8), (s, 0.02, 0.2), (r, 0.1, 0.9)):
        assert (a.astype(np.float32).astype(np.float64) == a).all()
        assert a.min() >= lo and a.max() <= hi


def test_view_sharding():
    for K, N in ((100, 8), (50, 4), (7, 3), (3, 8)):
        parts = [shard_views(K, N, r) for r in range(N)]
        assert sum(parts, []) == list(range(K))
    assert weak_views(50, 2) == list(range(100, 150))
    assert laplacian_weight(0) == 1.0 and laplacian_weight(3) == 0.0
