"""self_intersects / triangles_intersect (mesh.cpp:137-214).

Chain of pins: reference (oracle/_ref) -> tests/golden/selfint.npz -> oracle
(C brute force) -> GPU (cdr_self_intersects, LBVH). The answer is exact: the
bool and the full set of offending pairs (f < g) must be identical; pairs are
compared sorted by (f, g) (the reference's own order follows its BVH).

Finding: the reference test "coplanar overlap" (test_bvh.cpp:78-79) fails
against the reference itself: with tol = 1e-10 the shared normal axis has gap
0 > -tol |n|, which separates coplanar triangles, so the reference returns
False. The oracle and the GPU reproduce the reference, not the test.
"""
import os

import numpy as np
import pytest

from oracle.pyoracle import oracle_self_intersects, ref_self_intersects, triangles_intersect
from paper_2103_15208_b200 import scenes as S

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "selfint.npz")


def _cases():
    z = np.load(GOLD)
    return {str(n): (z[f"{n}_pos"], z[f"{n}_tris"], bool(z[f"{n}_result"]), z[f"{n}_pairs"]) for n in z["names"]}


CASES = sorted(_cases())
A = [(0, 0, 0), (1, 0, 0), (0, 1, 0)]
TRI_CASES = {  # test_bvh.cpp:71-82, with the reference's actual answers
    "crossing": ([(0.2, 0.2, -0.5), (0.4, 0.2, 0.5), (0.2, 0.4, 0.5)], True),
    "above": ([(0.2, 0.2, 0.5), (0.4, 0.2, 1.5), (0.2, 0.4, 1.5)], False),
    "coplanar_overlap": ([(0.1, 0.1, 0), (0.9, 0.1, 0), (0.1, 0.9, 0)], False),  # the test expects True
    "coplanar_disjoint": ([(2, 2, 0), (3, 2, 0), (2, 3, 0)], False),
}


def _tetrahedron(scale=0.5):  # make_tetrahedron (mesh.cpp:342-350)
    s = scale / np.sqrt(3.0)
    return (np.array([[s, s, s], [s, -s, -s], [-s, s, -s], [-s, -s, s]]),
            np.array([[0, 2, 1], [0, 1, 3], [0, 3, 2], [1, 2, 3]], np.int32))


# ---------------------------------------------------------------- oracle (CPU)
@pytest.mark.parametrize("name", CASES)
def test_oracle_matches_golden(name):
    pos, tris, res, pairs = _cases()[name]
    b, pr = oracle_self_intersects(pos, tris)
    assert b == res
    np.testing.assert_array_equal(pr, pairs)
    assert oracle_self_intersects(pos, tris, want_pairs=False)[0] == res


@pytest.mark.parametrize("case", sorted(TRI_CASES))
def test_oracle_triangles_intersect(case):
    b, want = TRI_CASES[case]
    assert triangles_intersect(A, b) == want


@pytest.mark.ref
@pytest.mark.parametrize("case", sorted(TRI_CASES))
def test_reference_triangles_intersect(case):
    b, want = TRI_CASES[case]
    assert triangles_intersect(A, b, ref=True) == want


def test_reference_unit_cases_restated():
    """test_mesh.cpp:112-150 on the oracle."""
    assert not oracle_self_intersects(*_tetrahedron())[0]
    ico = S.icosphere(2)
    assert not oracle_self_intersects(ico.positions, ico.triangles)[0]
    m = S.icosphere(1)
    p = m.positions.copy()
    p[3] = -p[3] * 1.3
    base = oracle_self_intersects(p, m.triangles)[0]
    assert oracle_self_intersects(p, m.triangles[::-1].copy())[0] == base  # reorder
    c, s = np.cos(0.7), np.sin(0.7)
    q = np.stack([c * p[:, 0] - s * p[:, 1], s * p[:, 0] + c * p[:, 1], p[:, 2]], 1) + np.array([5, -2, 3.0])
    assert oracle_self_intersects(q, m.triangles)[0] == base  # rigid transform


@pytest.mark.ref
def test_oracle_matches_reference_random():
    rng = np.random.default_rng(4)
    m = S.geodesic_sphere(8)
    for sd in (0.005, 0.02, 0.05):
        pos = m.positions + rng.normal(0, sd, m.positions.shape)
        a, b = oracle_self_intersects(pos, m.triangles), ref_self_intersects(pos, m.triangles)
        assert a[0] == b[0]
        np.testing.assert_array_equal(a[1], b[1])


# ---------------------------------------------------------------- GPU
def _renderer():
    from paper_2103_15208_b200.api import Renderer
    sc = S.make_scene(S.icosphere(1), 4, 1, 8)
    return Renderer(0, sc)


@pytest.mark.gpu
def test_gpu_matches_golden():
    r = _renderer()
    for name in CASES:
        pos, tris, res, pairs = _cases()[name]
        b, pr = r.self_intersects(pos, tris, want_pairs=True)
        assert b == res, name
        np.testing.assert_array_equal(pr, pairs, err_msg=name)
        assert r.self_intersects(pos, tris)[0] == res, name  # early-exit path


@pytest.mark.gpu
def test_gpu_unit_cases_and_topology_cache():
    r = _renderer()
    assert not r.self_intersects(*_tetrahedron())[0]
    m = S.icosphere(1)
    p = m.positions.copy()
    p[3] = -p[3] * 1.3
    base, pairs = oracle_self_intersects(p, m.triangles)
    # alternate topologies and positions: the cached topology must follow
    for tris in (m.triangles, m.triangles[::-1].copy(), m.triangles):
        b, pr = r.self_intersects(p, tris, want_pairs=True)
        ob, opr = oracle_self_intersects(p, tris)
        assert b == ob == base
        np.testing.assert_array_equal(pr, opr)
    assert not r.self_intersects(m.positions, m.triangles)[0]
    # fewer than two triangles, and a non-manifold fan (three faces on one edge)
    assert not r.self_intersects(np.zeros((3, 3)), np.array([[0, 1, 2]], np.int32))[0]
    fan = np.array([[0, 0, 0], [1, 0, 0], [0.5, 1, 0], [0.5, -1, 0.2], [0.5, 0.3, 1.0]])
    ft = np.array([[0, 1, 2], [0, 1, 3], [0, 1, 4]], np.int32)
    assert r.self_intersects(fan, ft, want_pairs=True)[0] == oracle_self_intersects(fan, ft)[0]


@pytest.mark.gpu
def test_gpu_matches_oracle_noisy_blob():
    r = _renderer()
    rng = np.random.default_rng(9)
    m = S.blob(10)
    for sd in (0.002, 0.008, 0.02):
        pos = m.positions + rng.normal(0, sd, m.positions.shape)
        b, pr = r.self_intersects(pos, m.triangles, want_pairs=True)
        ob, opr = oracle_self_intersects(pos, m.triangles)
        assert b == ob
        np.testing.assert_array_equal(pr, opr)
