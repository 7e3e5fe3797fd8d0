"""ctypes bindings to the two CPU checkers. TEST INFRASTRUCTURE ONLY.

* ``Oracle`` — the C restatement in oracle/cdr_oracle.c (kind "port").
* ``RefLib`` — the reference library compiled from its own unmodified sources
  (oracle/refbuild -> oracle/_ref/libcollodiff_ref.so, kind "reference").

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
reference leg may import this module; the product path never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libcdr_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libcollodiff_ref.so")
REFERENCE_SRC = "/root/reference/proj"

_d = C.POINTER(C.c_double)
_i = C.POINTER(C.c_int32)
_u64 = C.POINTER(C.c_uint64)
_vp = C.c_void_p


def build_oracle(force=False):
    if force or not os.path.exists(ORACLE_SO):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return ORACLE_SO


def build_ref(force=False):
    """Compile oracle/_ref from /root/reference (only where it exists)."""
    if os.path.exists(REF_SO) and not force:
        return REF_SO
    if not os.path.isdir(REFERENCE_SRC):
        return None
    subprocess.run(["make", "-s", "-j8", "-C", os.path.join(HERE, "refbuild")], check=True)
    return REF_SO


def ref_available():
    return os.path.exists(REF_SO) or os.path.isdir(REFERENCE_SRC)


def dp(a):
    return a.ctypes.data_as(_d) if a is not None else None


def ip(a):
    return a.ctypes.data_as(_i) if a is not None else None


class cdr_camera(C.Structure):
    _fields_ = [("origin", C.c_double * 3), ("right", C.c_double * 3), ("up", C.c_double * 3),
                ("forward", C.c_double * 3), ("fov_deg", C.c_double), ("width", C.c_int32),
                ("height", C.c_int32)]


class cdr_settings(C.Structure):
    _fields_ = [("spp", C.c_int32), ("boundary_term", C.c_int32),
                ("boundary_samples", C.c_int32), ("reserved", C.c_int32),
                ("seed", C.c_uint64), ("gamma", C.c_double)]


class cdr_layout(C.Structure):
    _fields_ = [("positions", C.c_int64), ("diffuse", C.c_int64), ("specular", C.c_int64),
                ("roughness", C.c_int64), ("light", C.c_int64), ("total", C.c_int64)]


SEGMENT_DTYPE = np.dtype([("v0", "<i4"), ("v1", "<i4"), ("p0", "<f8", 3), ("p1", "<f8", 3),
                          ("t0", "<f8"), ("t1", "<f8"), ("q0", "<f8", 2), ("q1", "<f8", 2),
                          ("z0", "<f8"), ("z1", "<f8"), ("length_px", "<f8")])
assert SEGMENT_DTYPE.itemsize == 128


class orc_scene(C.Structure):
    _fields_ = [("nv", C.c_int32), ("nt", C.c_int32), ("ne", C.c_int32),
                ("pos", _d), ("tris", _i), ("uv", _d), ("edges", _i),
                ("tw", C.c_int32), ("th", C.c_int32),
                ("diffuse", _d), ("specular", _d), ("roughness", _d),
                ("light", C.c_double * 3), ("background", C.c_double * 3),
                ("nviews", C.c_int32), ("cams", _vp), ("view_ids", _i)]


def layout_for(scene, optimize_light=False):
    """ParamLayout::for_scene (params.cpp:30-43)."""
    V = scene.mesh.V
    tw, th = scene.tex_res
    n = tw * th
    off = 0
    lay = {}
    for name, size in (("positions", 3 * V), ("diffuse", 3 * n), ("specular", 3 * n),
                       ("roughness", n)):
        lay[name] = off
        off += size
    lay["light"] = off if optimize_light else -1
    if optimize_light:
        off += 3
    lay["total"] = off
    return lay


def c_layout(lay):
    return cdr_layout(lay["positions"], lay["diffuse"], lay["specular"], lay["roughness"],
                      lay["light"], lay["total"])


def settings(spp, seed, gamma=2.2, boundary_term=1, boundary_samples=0):
    return cdr_settings(spp, boundary_term, boundary_samples, 0, seed, gamma)


def _cams(scene):
    from paper_2103_15208_b200.scenes import camera_struct_array
    return np.ascontiguousarray(camera_struct_array(scene.cameras))


class _SceneArrays:
    """Keeps contiguous copies alive for the C side."""

    def __init__(self, scene, view_ids=None):
        m = scene.mesh
        self.pos = np.ascontiguousarray(m.positions, dtype=np.float64)
        self.tris = np.ascontiguousarray(m.triangles, dtype=np.int32)
        self.uv = np.ascontiguousarray(m.uvs, dtype=np.float64)
        self.edges = np.ascontiguousarray(m.edges, dtype=np.int32)
        self.diffuse = np.ascontiguousarray(scene.diffuse, dtype=np.float64)
        self.specular = np.ascontiguousarray(scene.specular, dtype=np.float64)
        self.rough = np.ascontiguousarray(scene.roughness, dtype=np.float64)
        self.light = np.asarray(scene.light, dtype=np.float64)
        self.bg = np.asarray(scene.background, dtype=np.float64)
        self.cams = _cams(scene)
        self.view_ids = None if view_ids is None else np.ascontiguousarray(view_ids, dtype=np.int32)
        self.tw, self.th = scene.tex_res


def _self_intersects(fn, pos, tris, want_pairs):
    pos = np.ascontiguousarray(pos, dtype=np.float64)
    tris = np.ascontiguousarray(tris, dtype=np.int32)
    res = C.c_int32()
    n = C.c_int64()
    if not want_pairs:
        rc = fn(dp(pos), len(pos), ip(tris), len(tris), C.byref(res), None, C.c_int64(0), None)
        return bool(res.value), None, rc
    cap = max(16, 4 * len(tris))
    pairs = np.zeros((cap, 2), np.int32)
    rc = fn(dp(pos), len(pos), ip(tris), len(tris), C.byref(res), ip(pairs), C.c_int64(cap), C.byref(n))
    if rc == 0 and n.value > cap:
        cap = n.value
        pairs = np.zeros((cap, 2), np.int32)
        rc = fn(dp(pos), len(pos), ip(tris), len(tris), C.byref(res), ip(pairs), C.c_int64(cap), C.byref(n))
    return bool(res.value), pairs[:n.value].copy(), rc


def oracle_self_intersects(pos, tris, want_pairs=True):
    """self_intersects (mesh.cpp:184-214), C restatement: (bool, pairs sorted by (f, g))."""
    L = C.CDLL(build_oracle())
    b, pr, rc = _self_intersects(L.orc_self_intersects, pos, tris, want_pairs)
    assert rc == 0
    return b, pr


def ref_self_intersects(pos, tris, want_pairs=True):
    """The reference's own self_intersects (oracle/_ref), pairs sorted by (f, g)."""
    L = C.CDLL(build_ref())
    b, pr, rc = _self_intersects(L.ref_self_intersects, pos, tris, want_pairs)
    if rc != 0:
        raise RuntimeError(f"reference status {rc}")
    return b, pr


def triangles_intersect(a, b, tol=1e-10, ref=False):
    """triangles_intersect (mesh.cpp:160-182) of two 3x3 vertex arrays."""
    L = C.CDLL(build_ref() if ref else build_oracle())
    fn = L.ref_triangles_intersect if ref else L.orc_triangles_intersect
    fn.argtypes = [C.POINTER(C.c_double)] * 6 + [C.c_double]
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    return bool(fn(*(dp(np.ascontiguousarray(x)) for x in (a[0], a[1], a[2], b[0], b[1], b[2])), tol))


def adam_step(cfg, lay, nv, tex_wh, step, m, v, params, grad, ref=False):
    """adam_step (adam.cpp:9-54): oracle (C) or the reference itself. cfg =
    (beta1, beta2, epsilon, lr_positions, lr_textures, lr_light). Returns
    (status, step, m, v, params_out, displacement V x 3)."""
    m, v = np.array(m, dtype=np.float64), np.array(v, dtype=np.float64)
    out, disp = np.zeros(lay["total"]), np.zeros((nv, 3))
    st = C.c_int64(step)
    cf = np.asarray(cfg, dtype=np.float64)
    pr, gr = np.ascontiguousarray(params, dtype=np.float64), np.ascontiguousarray(grad, dtype=np.float64)
    if ref:
        L = C.CDLL(build_ref())
        rc = L.ref_adam_step(dp(cf), nv, tex_wh[0], tex_wh[1], int(lay["light"] >= 0), C.byref(st), dp(m), dp(v),
                             dp(pr), dp(gr), dp(out), dp(disp))
    else:
        L = C.CDLL(build_oracle())
        cl = c_layout(lay)
        rc = L.orc_adam_step(dp(cf), C.byref(cl), C.c_int64(nv), C.c_int64(tex_wh[0] * tex_wh[1]), C.byref(st),
                             dp(m), dp(v), dp(pr), dp(gr), dp(out), dp(disp))
    return rc, st.value, m, v, out, disp


def robust_evolve(pos, tris, disp, ref=False):
    """robust_evolve (evolve.cpp:19-53): (status, positions, applied scale)."""
    L = C.CDLL(build_ref() if ref else build_oracle())
    fn = L.ref_robust_evolve if ref else L.orc_robust_evolve
    pos = np.ascontiguousarray(pos, dtype=np.float64)
    tris = np.ascontiguousarray(tris, dtype=np.int32)
    d = np.ascontiguousarray(disp, dtype=np.float64)
    out = np.zeros_like(pos)
    sc = C.c_double()
    rc = fn(dp(pos), len(pos), ip(tris), len(tris), dp(d), dp(out), C.byref(sc))
    return rc, out, sc.value


def closest_points(pos, tris, queries, ref=False):
    """Bvh::closest_point (bvh.cpp:267-329) per query: oracle (brute force,
    ties to the lowest index) or the reference. (tri, point, dist, bary)."""
    L = C.CDLL(build_ref() if ref else build_oracle())
    fn = L.ref_closest_points if ref else L.orc_closest_points
    pos = np.ascontiguousarray(pos, dtype=np.float64)
    tris = np.ascontiguousarray(tris, dtype=np.int32)
    q = np.ascontiguousarray(queries, dtype=np.float64)
    n = len(q)
    tri, pt, di, ba = np.zeros(n, np.int32), np.zeros((n, 3)), np.zeros(n), np.zeros((n, 3))
    rc = fn(dp(pos), len(pos), ip(tris), len(tris), dp(q), n, ip(tri), dp(pt), dp(di), dp(ba))
    assert rc == 0
    return tri, pt, di, ba


def ref_point_to_mesh(pos, tris, queries):
    L = C.CDLL(build_ref())
    out = C.c_double()
    q = np.ascontiguousarray(queries, dtype=np.float64)
    rc = L.ref_point_to_mesh(dp(np.ascontiguousarray(pos, dtype=np.float64)), len(pos),
                             ip(np.ascontiguousarray(tris, dtype=np.int32)), len(tris), dp(q), len(q), C.byref(out))
    assert rc == 0
    return out.value


def ref_uv_transfer(old_pos, old_tris, old_uv, new_pos, max_distance):
    """(status, uvs) of uv_transfer (remesh.cpp:281-294)."""
    L = C.CDLL(build_ref())
    L.ref_uv_transfer.argtypes = [_vp, C.c_int32, _vp, C.c_int32, _vp, _vp, C.c_int32, C.c_double, _vp]
    op = np.ascontiguousarray(old_pos, dtype=np.float64)
    ot = np.ascontiguousarray(old_tris, dtype=np.int32)
    ou = np.ascontiguousarray(old_uv, dtype=np.float64)
    npos = np.ascontiguousarray(new_pos, dtype=np.float64)
    uv = np.zeros((len(npos), 2))
    rc = L.ref_uv_transfer(op.ctypes.data, len(op), ot.ctypes.data, len(ot), ou.ctypes.data, npos.ctypes.data,
                           len(npos), max_distance, uv.ctypes.data)
    return rc, uv


def _regularisers(fn, handle, scene, w, chk):
    V, n = scene.mesh.V, scene.diffuse.shape[0] * scene.diffuse.shape[1]
    vals = np.zeros(4)
    gp, gd, gs, gr = np.zeros((V, 3)), np.zeros((n, 3)), np.zeros((n, 3)), np.zeros(n)
    chk(fn(handle, dp(np.asarray(w, dtype=np.float64)), dp(vals), dp(gp), dp(gd), dp(gs), dp(gr)))
    return vals, gp, gd, gs, gr


class Oracle:
    """C restatement (oracle/cdr_oracle.c) over one scene."""

    def __init__(self, scene, view_ids=None):
        self.lib = C.CDLL(build_oracle())
        L = self.lib
        L.orc_ctx_new.restype = _vp
        L.orc_t_min.restype = C.c_double
        L.orc_last_error.restype = C.c_char_p
        self.scene = scene
        a = self.a = _SceneArrays(scene, view_ids)
        s = orc_scene()
        s.nv, s.nt, s.ne = scene.mesh.V, scene.mesh.T, scene.mesh.E
        s.pos, s.tris, s.uv, s.edges = dp(a.pos), ip(a.tris), dp(a.uv), ip(a.edges)
        s.tw, s.th = a.tw, a.th
        s.diffuse, s.specular, s.roughness = dp(a.diffuse), dp(a.specular), dp(a.rough)
        s.light = (C.c_double * 3)(*a.light)
        s.background = (C.c_double * 3)(*a.bg)
        s.nviews = len(scene.cameras)
        s.cams = a.cams.ctypes.data
        s.view_ids = ip(a.view_ids)
        self.s = s
        self.ctx = L.orc_ctx_new(C.byref(s))

    def __del__(self):
        try:
            self.lib.orc_ctx_free(C.c_void_p(self.ctx))
        except Exception:
            pass

    def _chk(self, rc):
        if rc != 0:
            raise RuntimeError(f"oracle status {rc}: {self.lib.orc_last_error().decode()}")

    @property
    def t_min(self):
        return self.lib.orc_t_min(C.c_void_p(self.ctx))

    def vertex_normals(self):
        out = np.zeros((self.scene.mesh.V, 3))
        self.lib.orc_vertex_normals(C.byref(self.s), dp(out))
        return out

    def intersect(self, orig, dirs, t_min=-1.0, brute=False):
        orig = np.ascontiguousarray(orig, dtype=np.float64)
        dirs = np.ascontiguousarray(dirs, dtype=np.float64)
        n = len(dirs)
        tri = np.zeros(n, np.int32)
        t, b1, b2 = np.zeros(n), np.zeros(n), np.zeros(n)
        fn = self.lib.orc_intersect_brute if brute else self.lib.orc_intersect
        fn(C.c_void_p(self.ctx), n, dp(orig), dp(dirs), C.c_double(t_min), ip(tri), dp(t), dp(b1), dp(b2))
        return tri, t, b1, b2

    def render(self, view, spp, seed):
        cam = self.scene.cameras[view]
        W, H = cam.width, cam.height
        rgb = np.zeros((H, W, 3))
        mask = np.zeros((H, W))
        hit = np.zeros(W * H * max(1, spp), np.int32)
        self._chk(self.lib.orc_render(C.c_void_p(self.ctx), view, spp, C.c_uint64(seed), dp(rgb), dp(mask), ip(hit)))
        return rgb, mask, hit

    def radiance_at(self, view, xy):
        xy = np.ascontiguousarray(xy, dtype=np.float64)
        rgb = np.zeros((len(xy), 3))
        tri = np.zeros(len(xy), np.int32)
        self.lib.orc_radiance_at(C.c_void_p(self.ctx), view, len(xy), dp(xy), dp(rgb), ip(tri))
        return rgb, tri

    def view_loss(self, rendered, target, target_mask=None, lam=1.0, gamma=2.2, use_mask=False):
        H, W = rendered.shape[:2]
        adj = np.zeros((H, W, 3))
        v = C.c_double()
        self.lib.orc_view_loss(W, H, dp(np.ascontiguousarray(rendered)), dp(np.ascontiguousarray(target)),
                               dp(None if target_mask is None else np.ascontiguousarray(target_mask)),
                               C.c_double(lam), C.c_double(gamma), int(use_mask), C.byref(v), dp(adj))
        return v.value, adj

    def interior(self, view, adjoint, spp, seed, hit, lay, grad=None):
        g = np.zeros(lay["total"]) if grad is None else grad
        cl = c_layout(lay)
        self._chk(self.lib.orc_interior(C.c_void_p(self.ctx), view, dp(np.ascontiguousarray(adjoint)), spp,
                                        C.c_uint64(seed), ip(np.ascontiguousarray(hit, dtype=np.int32)),
                                        C.byref(cl), dp(g)))
        return g

    def silhouettes(self, view):
        n = C.c_int32()
        tot = C.c_double()
        self.lib.orc_silhouettes(C.c_void_p(self.ctx), view, None, 0, C.byref(n), C.byref(tot))
        out = np.zeros(n.value, SEGMENT_DTYPE)
        self.lib.orc_silhouettes(C.c_void_p(self.ctx), view, out.ctypes.data_as(_vp), n.value,
                                 C.byref(n), C.byref(tot))
        return out, tot.value

    def boundary(self, view, adjoint, samples, seed, lay, probe=0, grad=None, segments=None):
        """boundary_pass; `segments` (SEGMENT_DTYPE) = a caller's SilhouetteSet,
        else this view's own extract_silhouettes."""
        g = np.zeros(lay["total"]) if grad is None else grad
        cl = c_layout(lay)
        deg = C.c_int32()
        if segments is not None:
            sg = np.ascontiguousarray(segments, dtype=SEGMENT_DTYPE)
            tot = 0.0
            for x in sg["length_px"]:  # silhouette.cpp:103
                tot += float(x)
            self._chk(self.lib.orc_boundary_segs(C.c_void_p(self.ctx), view, dp(np.ascontiguousarray(adjoint)),
                                                 sg.ctypes.data_as(C.c_void_p), len(sg), C.c_double(tot), samples,
                                                 C.c_uint64(seed), probe, C.byref(cl), dp(g), C.byref(deg)))
            return g, deg.value
        self._chk(self.lib.orc_boundary(C.c_void_p(self.ctx), view, dp(np.ascontiguousarray(adjoint)),
                                        samples, C.c_uint64(seed), probe, C.byref(cl), dp(g), C.byref(deg)))
        return g, deg.value

    def laplacian(self, mode=0, lam=0.1):
        V, E = self.scene.mesh.V, self.scene.mesh.E
        nnz = V + 2 * E
        outer = np.zeros(V + 1, np.int32)
        inner = np.zeros(nnz, np.int32)
        vals = np.zeros(nnz)
        grad = np.zeros((V, 3))
        v = C.c_double()
        self.lib.orc_laplacian(C.byref(self.s), mode, C.c_double(lam), C.byref(v), dp(grad),
                               ip(outer), ip(inner), dp(vals))
        return v.value, grad, (outer, inner, vals)

    def regularisers(self, w):
        """(values[4], grad_pos V x 3, grad_d, grad_s tex x 3, grad_r tex) of
        normal / edge / spec / roug; w = (normal, edge, spec, roug, sigma1, sigma2)."""
        return _regularisers(self.lib.orc_regularisers, C.byref(self.s), self.scene, w, self._chk)

    def loss_grad(self, targets_rgb, st, lay, lam_rend=1.0, lam_lap=0.1, lap_mode=0,
                  targets_mask=None, use_mask=False, want_rendered=False):
        g = np.zeros(lay["total"])
        loss = np.zeros(2)
        cl = c_layout(lay)
        tr = np.ascontiguousarray(targets_rgb, dtype=np.float64)
        rend = np.zeros_like(tr) if want_rendered else None
        self._chk(self.lib.orc_loss_grad(C.c_void_p(self.ctx), dp(tr),
                                         dp(None if targets_mask is None else np.ascontiguousarray(targets_mask)),
                                         C.byref(st), C.c_double(lam_rend), C.c_double(lam_lap), lap_mode,
                                         int(use_mask), C.byref(cl), dp(loss), dp(g), dp(rend)))
        return loss, g, rend


class RefLib:
    """The reference library itself (oracle/_ref), scene-bound."""

    def __init__(self, scene):
        so = build_ref()
        if so is None or not os.path.exists(so):
            raise FileNotFoundError("oracle/_ref not built and /root/reference absent")
        self.lib = L = C.CDLL(so)
        L.ref_last_error.restype = C.c_char_p
        L.ref_default_t_min.restype = C.c_double
        L.ref_tone_map.restype = C.c_double
        L.ref_tone_map_derivative.restype = C.c_double
        L.ref_tone_map.argtypes = [C.c_double, C.c_double]
        L.ref_tone_map_derivative.argtypes = [C.c_double, C.c_double]
        self.scene = scene
        a = self.a = _SceneArrays(scene)
        h = C.c_void_p()
        m = scene.mesh
        self._chk(L.ref_scene_new(dp(a.pos), m.V, ip(a.tris), m.T, dp(a.uv), dp(a.diffuse), dp(a.specular),
                                  dp(a.rough), a.tw, a.th, dp(a.light), dp(a.bg), a.cams.ctypes.data_as(_vp),
                                  len(scene.cameras), C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            self.lib.ref_scene_free(self.h)
        except Exception:
            pass

    def _chk(self, rc):
        if rc != 0:
            raise RuntimeError(f"reference status {rc}: {self.lib.ref_last_error().decode()}")

    def set_positions(self, pos):
        self.lib.ref_set_positions(self.h, dp(np.ascontiguousarray(pos, dtype=np.float64)))

    def edges(self):
        n = self.lib.ref_edge_count(self.h)
        out = np.zeros((n, 4), np.int32)
        self.lib.ref_edges(self.h, ip(out))
        return out

    @property
    def t_min(self):
        return self.lib.ref_default_t_min(self.h)

    def vertex_normals(self):
        out = np.zeros((self.scene.mesh.V, 3))
        self._chk(self.lib.ref_vertex_normals(self.h, dp(out)))
        return out

    def intersect(self, orig, dirs, t_min=-1.0):
        orig = np.ascontiguousarray(orig, dtype=np.float64)
        dirs = np.ascontiguousarray(dirs, dtype=np.float64)
        n = len(dirs)
        tri = np.zeros(n, np.int32)
        t, b1, b2 = np.zeros(n), np.zeros(n), np.zeros(n)
        self._chk(self.lib.ref_intersect(self.h, n, dp(orig), dp(dirs), C.c_double(t_min), ip(tri), dp(t),
                                         dp(b1), dp(b2)))
        return tri, t, b1, b2

    def render(self, view, spp, seed, threads=1):
        cam = self.scene.cameras[view]
        W, H = cam.width, cam.height
        rgb = np.zeros((H, W, 3))
        mask = np.zeros((H, W))
        hit = np.zeros(W * H * max(1, spp), np.int32)
        self._chk(self.lib.ref_render(self.h, view, spp, C.c_uint64(seed), threads, dp(rgb), dp(mask), ip(hit)))
        return rgb, mask, hit

    def radiance_at(self, view, xy):
        xy = np.ascontiguousarray(xy, dtype=np.float64)
        rgb = np.zeros((len(xy), 3))
        tri = np.zeros(len(xy), np.int32)
        self._chk(self.lib.ref_radiance_at(self.h, view, len(xy), dp(xy), dp(rgb), ip(tri)))
        return rgb, tri

    def view_loss(self, rendered, target, target_mask=None, lam=1.0, gamma=2.2, use_mask=False):
        H, W = rendered.shape[:2]
        adj = np.zeros((H, W, 3))
        v = C.c_double()
        self._chk(self.lib.ref_view_loss(W, H, dp(np.ascontiguousarray(rendered)), dp(np.ascontiguousarray(target)),
                                         dp(None if target_mask is None else np.ascontiguousarray(target_mask)),
                                         C.c_double(lam), C.c_double(gamma), int(use_mask), C.byref(v), dp(adj)))
        return v.value, adj

    def interior(self, view, adjoint, spp, seed, hit, lay, threads=1, grad=None):
        g = np.zeros(lay["total"]) if grad is None else grad
        hit = np.ascontiguousarray(hit, dtype=np.int32)
        self._chk(self.lib.ref_interior(self.h, view, dp(np.ascontiguousarray(adjoint)), spp, C.c_uint64(seed),
                                        threads, ip(hit), C.c_int64(len(hit)), int(lay["light"] >= 0), dp(g)))
        return g

    def silhouettes(self, view):
        n = C.c_int32()
        tot = C.c_double()
        self._chk(self.lib.ref_silhouettes(self.h, view, None, 0, C.byref(n), C.byref(tot)))
        out = np.zeros(n.value, SEGMENT_DTYPE)
        self._chk(self.lib.ref_silhouettes(self.h, view, out.ctypes.data_as(_vp), n.value, C.byref(n),
                                           C.byref(tot)))
        return out, tot.value

    def boundary(self, view, adjoint, samples, seed, lay, probe=0, grad=None):
        g = np.zeros(lay["total"]) if grad is None else grad
        deg = C.c_int32()
        self._chk(self.lib.ref_boundary(self.h, view, dp(np.ascontiguousarray(adjoint)), samples,
                                        C.c_uint64(seed), probe, int(lay["light"] >= 0), dp(g), C.byref(deg)))
        return g, deg.value

    def laplacian(self, mode=0, lam=0.1):
        V = self.scene.mesh.V
        nnz = C.c_int64()
        self._chk(self.lib.ref_laplacian(self.h, mode, C.c_double(lam), None, None, None, None, None,
                                         C.byref(nnz)))
        outer = np.zeros(V + 1, np.int32)
        inner = np.zeros(nnz.value, np.int32)
        vals = np.zeros(nnz.value)
        grad = np.zeros((V, 3))
        v = C.c_double()
        self._chk(self.lib.ref_laplacian(self.h, mode, C.c_double(lam), C.byref(v), dp(grad), ip(outer),
                                         ip(inner), dp(vals), C.byref(nnz)))
        return v.value, grad, (outer, inner, vals)

    def regularisers(self, w):
        return _regularisers(self.lib.ref_regularisers, self.h, self.scene, w, self._chk)

    def total_loss(self, targets_rgb, spp, seed, lay, threads=1, lam_rend=1.0, lam_lap=0.1,
                   boundary_term=1, boundary_samples=0, gamma=2.2, lap_mode=0,
                   others=(0.0, 0.0, 0.0, 0.0), targets_mask=None, use_mask=False, want_rendered=False):
        g = np.zeros(lay["total"])
        bd = np.zeros(7)
        w = np.array([lam_rend, lam_lap, *others], dtype=np.float64)
        tr = np.ascontiguousarray(targets_rgb, dtype=np.float64)
        rend = np.zeros_like(tr) if want_rendered else None
        self._chk(self.lib.ref_total_loss(self.h, dp(tr),
                                          dp(None if targets_mask is None else np.ascontiguousarray(targets_mask)),
                                          spp, C.c_uint64(seed), threads, boundary_term, boundary_samples,
                                          C.c_double(gamma), dp(w), int(use_mask), lap_mode,
                                          int(lay["light"] >= 0), dp(g), dp(bd), dp(rend)))
        return bd, g, rend


def ref_primitives():
    """Unbound reference primitives (camera, RNG, BRDF, texture, tone map)."""
    so = build_ref()
    if so is None:
        raise FileNotFoundError("oracle/_ref unavailable")
    L = C.CDLL(so)
    L.ref_tone_map.restype = C.c_double
    L.ref_tone_map_derivative.restype = C.c_double
    L.ref_tone_map.argtypes = [C.c_double, C.c_double]
    L.ref_tone_map_derivative.argtypes = [C.c_double, C.c_double]
    return L


def oracle_primitives():
    return C.CDLL(build_oracle())
