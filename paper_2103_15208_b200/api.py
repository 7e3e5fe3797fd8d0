"""Python host mirror of the reference hot-path API over libcdr.so (ctypes).

The reference is a C++ library; its drop-in is the C-ABI in include/cdr.h
(see INTEGRATION.md for the C++ shim that defines the collodiff:: symbols on
top of it). This module is the same boundary seen from Python, used by the
tests, smoke() and bench.py. Names, argument meaning and error behaviour
follow the reference:

  Renderer.render             render           (render.hpp:67-68)
  Renderer.radiance_at        radiance_at      (render.hpp:61-62)
  Renderer.view_rendering_loss view_rendering_loss (losses.hpp:37-38)
  Renderer.interior_pass      interior_pass    (diff_render.hpp:48-50)
  Renderer.extract_silhouettes extract_silhouettes (silhouette.hpp:36)
  Renderer.boundary_pass      boundary_pass    (diff_render.hpp:56-59)
  Renderer.grad_image_loss    grad_image_loss  (diff_render.hpp:65-67)
  Renderer.total_loss         total_loss, hot subset (losses.hpp:94-96)
  Renderer.cotangent_laplacian / laplacian_loss (laplacian.hpp:14, losses.hpp:53)

Errors raise SizeMismatch / NonFiniteGradient / CollodiffError (errors.hpp).
There is no CPU fallback: without the built library or a CUDA device every
call raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from .scenes import CAMERA_DTYPE, Scene, camera_struct_array

LIB_PATH = os.environ.get("CDR_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libcdr.so")


class CollodiffError(RuntimeError):
    """collodiff::Error (errors.hpp:8-10)."""


class SizeMismatch(CollodiffError):
    """collodiff::SizeMismatch (errors.hpp:24-26)."""


class NonFiniteGradient(CollodiffError):
    """collodiff::NonFiniteGradient (errors.hpp:28-30)."""


class NoDevice(CollodiffError):
    pass


class InputSelfIntersecting(CollodiffError):
    """collodiff::InputSelfIntersecting (errors.hpp:32-34)."""


class ProjectionTooFar(CollodiffError):
    """collodiff::ProjectionTooFar (errors.hpp:40)."""


_d = C.POINTER(C.c_double)
_i = C.POINTER(C.c_int32)
_vp = C.c_void_p


class cdr_settings(C.Structure):
    _fields_ = [("spp", C.c_int32), ("boundary_term", C.c_int32), ("boundary_samples", C.c_int32),
                ("flags", C.c_int32), ("seed", C.c_uint64), ("gamma", C.c_double)]


class cdr_layout(C.Structure):
    _fields_ = [("positions", C.c_int64), ("diffuse", C.c_int64), ("specular", C.c_int64),
                ("roughness", C.c_int64), ("light", C.c_int64), ("total", C.c_int64)]


CDR_FLAG_GRAD_OVERWRITE = 1


class cdr_adam_config(C.Structure):
    _fields_ = [("beta1", C.c_double), ("beta2", C.c_double), ("epsilon", C.c_double),
                ("lr_positions", C.c_double), ("lr_textures", C.c_double), ("lr_light", C.c_double)]


class cdr_reg_weights(C.Structure):
    _fields_ = [("normal", C.c_double), ("edge", C.c_double), ("spec", C.c_double), ("roug", C.c_double),
                ("sigma1", C.c_double), ("sigma2", C.c_double)]


class cdr_stats(C.Structure):
    _fields_ = [("pixels", C.c_int64), ("samples", C.c_int64), ("hit_samples", C.c_int64),
                ("adjoint_samples", C.c_int64), ("boundary_samples", C.c_int64),
                ("boundary_active", C.c_int64), ("segments", C.c_int64),
                ("degenerate_skipped", C.c_int32), ("nonfinite", C.c_int32),
                ("ms_prepare", C.c_double), ("ms_render", C.c_double), ("ms_silhouette", C.c_double),
                ("ms_boundary", C.c_double), ("ms_finalize", C.c_double), ("ms_total", C.c_double),
                ("kernel_launches", C.c_int64), ("ms_trace", C.c_double), ("beam_fallback_tiles", C.c_int64),
                ("shaded_samples", C.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


SEGMENT_DTYPE = np.dtype([("v0", "<i4"), ("v1", "<i4"), ("p0", "<f8", 3), ("p1", "<f8", 3),
                          ("t0", "<f8"), ("t1", "<f8"), ("q0", "<f8", 2), ("q1", "<f8", 2),
                          ("z0", "<f8"), ("z1", "<f8"), ("length_px", "<f8")])

_ERRORS = {1: SizeMismatch, 2: NonFiniteGradient, 3: CollodiffError, 4: CollodiffError,
           5: CollodiffError, 6: NoDevice, 7: InputSelfIntersecting, 8: ProjectionTooFar}

_lib = None


ABI_VERSION = 2  # include/cdr.h CDR_ABI_VERSION


def load_library(path: str = LIB_PATH):
    """Load libcdr.so; raises if it was not built (no silent fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} missing: run `python -m paper_2103_15208_b200.build`")
    L = C.CDLL(path)
    if L.cdr_abi_version() != ABI_VERSION:  # the ctypes structs below follow this header version
        raise RuntimeError(f"{path}: ABI version {L.cdr_abi_version()}, this binding expects {ABI_VERSION}: rebuild")
    L.cdr_build_flags.restype = C.c_int
    L.cdr_last_error.restype = C.c_char_p
    L.cdr_last_error.argtypes = [_vp]
    L.cdr_create.argtypes = [C.c_int, C.POINTER(_vp)]
    L.cdr_destroy.argtypes = [_vp]
    L.cdr_destroy.restype = None
    L.cdr_get_stream.argtypes = [_vp, C.POINTER(_vp)]
    L.cdr_set_mesh.argtypes = [_vp, _d, C.c_int32, _i, C.c_int32, _d, _i, C.c_int32]
    L.cdr_update_positions.argtypes = [_vp, _d]
    L.cdr_get_edges.argtypes = [_vp, _i, _i]
    L.cdr_set_textures.argtypes = [_vp, _d, _d, _d, C.c_int32, C.c_int32]
    L.cdr_stage_params.argtypes = [_vp, _d, _d, _d, _d, C.c_int32, C.c_int32]
    L.cdr_set_light.argtypes = [_vp, _d, _d]
    L.cdr_set_views.argtypes = [_vp, _vp, _i, C.c_int32]
    L.cdr_set_target.argtypes = [_vp, C.c_int32, _d, _d]
    L.cdr_set_target_f32.argtypes = [_vp, C.c_int32, C.POINTER(C.c_float), C.POINTER(C.c_float)]
    L.cdr_vertex_normals.argtypes = [_vp, _d]
    L.cdr_render.argtypes = [_vp, C.c_int32, C.POINTER(cdr_settings), _d, _d, _i]
    L.cdr_radiance_at.argtypes = [_vp, C.c_int32, C.c_int32, _d, _d, _i]
    L.cdr_probe_points.argtypes = [_vp, C.c_int32, C.c_int32, _d, _d, _i]
    L.cdr_view_loss.argtypes = [_vp, C.c_int32, C.c_int32, _d, _d, _d, C.c_double, C.c_double, C.c_int32,
                                _d, _d]
    L.cdr_interior_pass.argtypes = [_vp, C.c_int32, _d, C.POINTER(cdr_settings), _i, C.c_int64,
                                    C.POINTER(cdr_layout), _d]
    L.cdr_extract_silhouettes.argtypes = [_vp, C.c_int32, _vp, C.c_int32, _i, _d]
    L.cdr_boundary_pass.argtypes = [_vp, C.c_int32, _d, _vp, C.c_int32, C.c_int32, C.c_uint64, C.c_int32,
                                    C.POINTER(cdr_layout), _d, _i]
    L.cdr_loss_grad.argtypes = [_vp, _i, C.c_int32, C.POINTER(cdr_settings), C.c_double, C.c_double,
                                C.c_int32, C.c_int32, C.POINTER(cdr_layout), _d, _d, _d, _d,
                                C.POINTER(cdr_stats)]
    L.cdr_total_loss.argtypes = [_vp, _i, C.c_int32, C.POINTER(cdr_settings), C.c_double, C.c_double,
                                 C.POINTER(cdr_reg_weights), C.c_int32, C.c_int32, C.POINTER(cdr_layout), _d, _d,
                                 _d, _d, C.POINTER(cdr_stats)]
    L.cdr_regularisers.argtypes = [_vp, C.POINTER(cdr_reg_weights), C.POINTER(cdr_layout), _d, _d]
    L.cdr_get_rendered.argtypes = [_vp, C.c_int32, _d, _d]
    L.cdr_lbvh_keys.argtypes = [_vp, C.POINTER(C.c_uint64), C.c_int32]
    L.cdr_closest_points.argtypes = [_vp, _d, C.c_int32, _i, C.c_int32, _d, C.c_int32, _i, _d, _d, _d]
    L.cdr_adam_init.argtypes = [_vp, C.POINTER(cdr_adam_config), C.POINTER(cdr_layout)]
    L.cdr_adam_step.argtypes = [_vp, _d, C.POINTER(C.c_int64)]
    L.cdr_adam_get_state.argtypes = [_vp, _d, _d, C.POINTER(C.c_int64)]
    L.cdr_adam_set_state.argtypes = [_vp, _d, _d, C.c_int64]
    L.cdr_evolve.argtypes = [_vp, _d, C.POINTER(C.c_double), _d]
    L.cdr_get_params.argtypes = [_vp, C.POINTER(cdr_layout), _d]
    L.cdr_self_intersects.argtypes = [_vp, _d, C.c_int32, _i, C.c_int32, _i, _i, C.c_int64,
                                      C.POINTER(C.c_int64)]
    L.cdr_get_grad.argtypes = [_vp, _d, C.c_int64]
    L.cdr_set_grad.argtypes = [_vp, _d, C.c_int64]
    L.cdr_grad_device_ptr.argtypes = [_vp, C.POINTER(_vp), C.POINTER(C.c_int64)]
    L.cdr_laplacian_matrix.argtypes = [_vp, C.c_int32, _i, _i, _d, C.POINTER(C.c_int64)]
    L.cdr_laplacian_loss.argtypes = [_vp, C.c_int32, C.c_double, _d, _d]
    L.cdr_nccl_unique_id.argtypes = [C.c_char_p]
    L.cdr_comm_init.argtypes = [_vp, C.c_char_p, C.c_int32, C.c_int32]
    L.cdr_comm_info.argtypes = [_vp, _i, _i]
    L.cdr_comm_init_all.argtypes = [C.POINTER(_vp), C.c_int32]
    L.cdr_set_rank.argtypes = [_vp, C.c_int32, C.c_int32]
    L.cdr_device_count.argtypes = [C.POINTER(C.c_int)]
    _lib = L
    return L


def exported_symbols():
    """Names declared in include/cdr.h (for the load/export test)."""
    import re
    hdr = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "cdr.h")
    src = open(hdr).read()
    return sorted(set(re.findall(r"\b(cdr_[a-z_0-9]+)\s*\(", src)))


def _dp(a):
    return None if a is None else a.ctypes.data_as(_d)


def _ip(a):
    return None if a is None else a.ctypes.data_as(_i)


@dataclass
class RenderSettings:
    """RenderSettings (render.hpp:27-35)."""
    spp: int = 4
    seed: int = 0
    gamma: float = 2.2
    boundary_term: bool = True
    boundary_samples: int = 0

    def c(self):
        return cdr_settings(int(self.spp), int(bool(self.boundary_term)), int(self.boundary_samples), 0,
                            int(self.seed) & (2 ** 64 - 1), float(self.gamma))


@dataclass
class LossWeights:
    """LossWeights (losses.hpp:14-23), the reference defaults."""
    rend: float = 1.0
    lap: float = 0.1
    normal: float = 0.01
    edge: float = 1.0
    spec: float = 0.01
    roug: float = 0.001
    sigma1: float = 2.0
    sigma2: float = 0.1

    def c_reg(self):
        return cdr_reg_weights(self.normal, self.edge, self.spec, self.roug, self.sigma1, self.sigma2)


@dataclass
class AdamConfig:
    """AdamConfig (optimize.hpp:13-18)."""
    beta1: float = 0.9
    beta2: float = 0.999
    epsilon: float = 1e-8
    lr_positions: float = 1e-3
    lr_textures: float = 1e-2
    lr_light: float = 1e-2

    def c(self):
        return cdr_adam_config(self.beta1, self.beta2, self.epsilon, self.lr_positions, self.lr_textures,
                               self.lr_light)

    def tuple(self):
        return (self.beta1, self.beta2, self.epsilon, self.lr_positions, self.lr_textures, self.lr_light)


def param_layout(scene: Scene, optimize_light: bool = False) -> dict:
    """ParamLayout::for_scene (params.cpp:30-43)."""
    tw, th = scene.tex_res
    n = tw * th
    lay, off = {}, 0
    for name, size in (("positions", 3 * scene.mesh.V), ("diffuse", 3 * n), ("specular", 3 * n),
                       ("roughness", n)):
        lay[name] = off
        off += size
    lay["light"] = off if optimize_light else -1
    off += 3 if optimize_light else 0
    lay["total"] = off
    return lay


def _clayout(lay):
    return cdr_layout(lay["positions"], lay["diffuse"], lay["specular"], lay["roughness"], lay["light"],
                      lay["total"])


class Renderer:
    """One GPU context (cdr_ctx) holding a scene: the GradContext equivalent."""

    def __init__(self, device: int = 0, scene: Scene | None = None, view_ids=None):
        self.L = load_library()
        h = _vp()
        rc = self.L.cdr_create(device, C.byref(h))
        if rc != 0:
            raise _ERRORS.get(rc, CollodiffError)(f"cdr_create failed with status {rc}")
        self.h = h
        self.scene = None
        if scene is not None:
            self.set_scene(scene, view_ids)

    def close(self):
        if getattr(self, "h", None):
            self.L.cdr_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _chk(self, rc):
        if rc != 0:
            msg = self.L.cdr_last_error(self.h).decode()
            raise _ERRORS.get(rc, CollodiffError)(msg)

    # ---------------------------------------------------------------- state
    def set_scene(self, scene: Scene, view_ids=None):
        self.scene = scene
        self.set_mesh(scene.mesh)
        self.set_textures(scene.diffuse, scene.specular, scene.roughness)
        self.set_light(scene.light, scene.background)
        self.set_views(scene.cameras, view_ids)

    def set_mesh(self, mesh):
        self._pos = np.ascontiguousarray(mesh.positions, dtype=np.float64)
        tris = np.ascontiguousarray(mesh.triangles, dtype=np.int32)
        uv = None if mesh.uvs is None else np.ascontiguousarray(mesh.uvs, dtype=np.float64)
        edges = None if mesh.edges is None else np.ascontiguousarray(mesh.edges, dtype=np.int32)
        self._chk(self.L.cdr_set_mesh(self.h, _dp(self._pos), len(self._pos), _ip(tris), len(tris), _dp(uv),
                                      _ip(edges), 0 if edges is None else len(edges)))
        self.V = len(self._pos)
        self.T = len(tris)

    def update_positions(self, pos):
        pos = np.ascontiguousarray(pos, dtype=np.float64)
        self._chk(self.L.cdr_update_positions(self.h, _dp(pos)))

    def edges(self):
        n = C.c_int32()
        self._chk(self.L.cdr_get_edges(self.h, None, C.byref(n)))
        out = np.zeros((n.value, 4), np.int32)
        self._chk(self.L.cdr_get_edges(self.h, _ip(out), C.byref(n)))
        return out

    def set_textures(self, diffuse, specular, roughness):
        d = np.ascontiguousarray(diffuse, dtype=np.float64)
        s = np.ascontiguousarray(specular, dtype=np.float64)
        r = np.ascontiguousarray(roughness, dtype=np.float64)
        h, w = r.shape[:2]
        self._chk(self.L.cdr_set_textures(self.h, _dp(d), _dp(s), _dp(r), w, h))

    def stage_params(self, positions=None, maps=None):
        """Parameters read by the next loss_grad / total_loss call
        (cdr_stage_params): positions (V x 3) and/or maps = (diffuse,
        specular, roughness). With pinned arrays the maps' upload and the
        gradient/image downloads overlap that call's kernels. The arrays are
        kept referenced here until then (the library reads them in the call)."""
        pos = None if positions is None else np.ascontiguousarray(positions, dtype=np.float64)
        d = s = r = None
        w = h = 0
        if maps is not None:
            if len(maps) != 3 or any(m is None for m in maps):
                raise ValueError("maps = (diffuse, specular, roughness), all three")
            d, s, r = (np.ascontiguousarray(m, dtype=np.float64) for m in maps)
            h, w = r.shape[:2]
        self._staged = (pos, d, s, r)
        self._chk(self.L.cdr_stage_params(self.h, _dp(pos), _dp(d), _dp(s), _dp(r), w, h))

    def set_light(self, intensity, background=(0.0, 0.0, 0.0)):
        a = np.asarray(intensity, dtype=np.float64)
        b = np.asarray(background, dtype=np.float64)
        self._chk(self.L.cdr_set_light(self.h, _dp(a), _dp(b)))

    def set_views(self, cameras, view_ids=None):
        self._cams = np.ascontiguousarray(camera_struct_array(cameras))
        ids = None if view_ids is None else np.ascontiguousarray(view_ids, dtype=np.int32)
        self._chk(self.L.cdr_set_views(self.h, self._cams.ctypes.data_as(_vp), _ip(ids), len(cameras)))
        self.cameras = list(cameras)

    def set_target(self, view, rgb, mask=None):
        """Target image (H x W x 3) and optional mask of a view slot; float32
        arrays (PFM data) take the fp32 upload path (cdr_set_target_f32)."""
        if np.asarray(rgb).dtype == np.float32:
            fp = C.POINTER(C.c_float)
            rgb = np.ascontiguousarray(rgb, dtype=np.float32)
            mask = None if mask is None else np.ascontiguousarray(mask, dtype=np.float32)
            self._chk(self.L.cdr_set_target_f32(self.h, view, rgb.ctypes.data_as(fp),
                                                None if mask is None else mask.ctypes.data_as(fp)))
            return
        rgb = np.ascontiguousarray(rgb, dtype=np.float64)
        mask = None if mask is None else np.ascontiguousarray(mask, dtype=np.float64)
        self._chk(self.L.cdr_set_target(self.h, view, _dp(rgb), _dp(mask)))

    def stream(self):
        s = _vp()
        self._chk(self.L.cdr_get_stream(self.h, C.byref(s)))
        return s.value

    # ---------------------------------------------------------------- reference API
    def vertex_normals(self):
        out = np.zeros((self.V, 3))
        self._chk(self.L.cdr_vertex_normals(self.h, _dp(out)))
        return out

    def render(self, view, settings: RenderSettings, want_hits=True):
        cam = self.cameras[view]
        W, H = cam.width, cam.height
        spp = max(1, settings.spp)
        rgb = np.zeros((H, W, 3))
        mask = np.zeros((H, W))
        hit = np.zeros(W * H * spp, np.int32) if want_hits else None
        st = settings.c()
        self._chk(self.L.cdr_render(self.h, view, C.byref(st), _dp(rgb), _dp(mask), _ip(hit)))
        return rgb, mask, hit

    def radiance_at(self, view, xy):
        xy = np.ascontiguousarray(xy, dtype=np.float64).reshape(-1, 2)
        rgb = np.zeros((len(xy), 3))
        tri = np.zeros(len(xy), np.int32)
        self._chk(self.L.cdr_radiance_at(self.h, view, len(xy), _dp(xy), _dp(rgb), _ip(tri)))
        return rgb, tri

    def probe_points(self, view, xy):
        """The boundary pass's radiance probes through the candidate lists of
        the last render / loss call (points traced in pairs, as one edge
        sample's x - n/2 and x + n/2): (rgb n x 3, tri n)."""
        xy = np.ascontiguousarray(xy, dtype=np.float64).reshape(-1, 2)
        rgb = np.zeros((len(xy), 3))
        tri = np.zeros(len(xy), np.int32)
        self._chk(self.L.cdr_probe_points(self.h, view, len(xy), _dp(xy), _dp(rgb), _ip(tri)))
        return rgb, tri

    def view_rendering_loss(self, rendered, target, lambda_rend=1.0, gamma=2.2, target_mask=None,
                            use_target_mask=False):
        rendered = np.ascontiguousarray(rendered, dtype=np.float64)
        target = np.ascontiguousarray(target, dtype=np.float64)
        if rendered.shape != target.shape:
            raise SizeMismatch("rendered/target size mismatch")
        H, W = rendered.shape[:2]
        adj = np.zeros((H, W, 3))
        v = C.c_double()
        tm = None if target_mask is None else np.ascontiguousarray(target_mask, dtype=np.float64)
        self._chk(self.L.cdr_view_loss(self.h, W, H, _dp(rendered), _dp(target), _dp(tm), lambda_rend, gamma,
                                       int(use_target_mask), C.byref(v), _dp(adj)))
        return v.value, adj

    def interior_pass(self, view, adjoint, settings: RenderSettings, hit_cache, layout, grad=None):
        g = np.zeros(layout["total"]) if grad is None else grad
        adjoint = np.ascontiguousarray(adjoint, dtype=np.float64)
        cam = self.cameras[view]
        if adjoint.shape[:2] != (cam.height, cam.width):
            raise SizeMismatch("adjoint size does not match view")
        hc = np.ascontiguousarray(hit_cache, dtype=np.int32)
        st = settings.c()
        lay = _clayout(layout)
        self._chk(self.L.cdr_interior_pass(self.h, view, _dp(adjoint), C.byref(st), _ip(hc), len(hc),
                                           C.byref(lay), _dp(g)))
        return g

    def extract_silhouettes(self, view):
        n = C.c_int32()
        tot = C.c_double()
        self._chk(self.L.cdr_extract_silhouettes(self.h, view, None, 0, C.byref(n), C.byref(tot)))
        out = np.zeros(n.value, SEGMENT_DTYPE)
        self._chk(self.L.cdr_extract_silhouettes(self.h, view, out.ctypes.data_as(_vp), n.value, C.byref(n),
                                                 C.byref(tot)))
        return out, tot.value

    def boundary_pass(self, view, adjoint, samples, seed, layout, segments=None, probe=0, grad=None):
        g = np.zeros(layout["total"]) if grad is None else grad
        adjoint = np.ascontiguousarray(adjoint, dtype=np.float64)
        cam = self.cameras[view]
        if adjoint.shape[:2] != (cam.height, cam.width):
            raise SizeMismatch("adjoint size does not match view")
        lay = _clayout(layout)
        deg = C.c_int32()
        segp, nseg = None, 0
        if segments is not None:
            segments = np.ascontiguousarray(segments, dtype=SEGMENT_DTYPE)
            segp, nseg = segments.ctypes.data_as(_vp), len(segments)
        self._chk(self.L.cdr_boundary_pass(self.h, view, _dp(adjoint), segp, nseg, samples, seed & (2 ** 64 - 1),
                                           probe, C.byref(lay), _dp(g), C.byref(deg)))
        return g, deg.value

    def loss_grad(self, views, settings: RenderSettings, layout, lambda_rend=1.0, lambda_lap=0.1,
                  laplacian_mode=0, use_target_mask=False, grad=None, want_rendered=False, device_only=False,
                  overwrite=False, rendered_out=None, mask_out=None):
        """Rendering + Laplacian part of total_loss over `views` (slots). Returns
        (loss[2], grad, stats, rendered). The gradient is added to `grad` (fresh
        zeros by default), or written over it with overwrite=True (the caller's
        buffer is then not read: CDR_FLAG_GRAD_OVERWRITE)."""
        views = np.ascontiguousarray(views, dtype=np.int32)
        st = settings.c()
        if overwrite:
            st.flags |= CDR_FLAG_GRAD_OVERWRITE
        lay = _clayout(layout)
        loss = np.zeros(2)
        g = None if device_only else (np.zeros(layout["total"]) if grad is None else grad)
        rend = rendered_out
        if want_rendered and rend is None:
            npx = sum(self.cameras[v].width * self.cameras[v].height for v in views)
            rend = np.zeros(3 * npx)
        stats = cdr_stats()
        self._chk(self.L.cdr_loss_grad(self.h, _ip(views), len(views), C.byref(st), lambda_rend, lambda_lap,
                                       laplacian_mode, int(use_target_mask), C.byref(lay), _dp(loss), _dp(g),
                                       _dp(rend), _dp(mask_out), C.byref(stats)))
        return loss, g, stats, rend

    def total_loss(self, targets, settings: RenderSettings, layout, lambda_rend=1.0, lambda_lap=0.1,
                   laplacian_mode=0, use_target_masks=False, target_masks=None, weights=None):
        """total_loss (losses.cpp:244-297): breakdown {total, rend, lap, normal,
        edge, spec, roug}, fresh gradient, rendered images. `weights`
        (LossWeights) gives every term its weight; without it the call keeps the
        lambda_rend / lambda_lap arguments and the four regularisers at zero."""
        if len(targets) != len(self.cameras):
            raise SizeMismatch("target count does not match views")
        for k, t in enumerate(targets):
            self.set_target(k, t, None if target_masks is None else target_masks[k])
        w = weights if weights is not None else LossWeights(lambda_rend, lambda_lap, 0.0, 0.0, 0.0, 0.0)
        views = np.arange(len(self.cameras), dtype=np.int32)
        st = settings.c()
        st.flags |= CDR_FLAG_GRAD_OVERWRITE  # a fresh GradVector (losses.cpp:250)
        lay = _clayout(layout)
        reg = w.c_reg()
        bd = np.zeros(7)
        g = np.empty(layout["total"])
        rend = np.zeros(sum(3 * c.width * c.height for c in self.cameras))
        stats = cdr_stats()
        self._chk(self.L.cdr_total_loss(self.h, _ip(views), len(views), C.byref(st), w.rend, w.lap, C.byref(reg),
                                        laplacian_mode, int(use_target_masks), C.byref(lay), _dp(bd), _dp(g),
                                        _dp(rend), None, C.byref(stats)))
        rendered, off = [], 0
        for cam in self.cameras:
            n = cam.width * cam.height * 3
            rendered.append(rend[off:off + n].reshape(cam.height, cam.width, 3))
            off += n
        keys = ("total", "rend", "lap", "normal", "edge", "spec", "roug")
        return dict(zip(keys, bd.tolist())), g, rendered

    def total_loss_device(self, views, settings: RenderSettings, layout, weights=None, laplacian_mode=0,
                          use_target_masks=False):
        """cdr_total_loss over `views` (slots) with the targets already set and
        the gradient left on the device (for adam_step): the resident form of
        total_loss. Returns (breakdown dict, stats)."""
        w = weights if weights is not None else LossWeights()
        views = np.ascontiguousarray(views, dtype=np.int32)
        st = settings.c()
        bd = np.zeros(7)
        stats = cdr_stats()
        self._chk(self.L.cdr_total_loss(self.h, _ip(views), len(views), C.byref(st), w.rend, w.lap,
                                        C.byref(w.c_reg()), laplacian_mode, int(use_target_masks),
                                        C.byref(_clayout(layout)), _dp(bd), None, None, None, C.byref(stats)))
        keys = ("total", "rend", "lap", "normal", "edge", "spec", "roug")
        return dict(zip(keys, bd.tolist())), stats

    def regularisers(self, weights, layout, grad=None, device_only=False):
        """normal_consistency / edge_length / specular_correlation / roughness_tv
        (losses.cpp:80-238). Returns ({normal, edge, spec, roug}, grad) with the
        gradients += into `grad` (ParamLayout order; fresh zeros by default), or
        into the device gradient with device_only (grad is then None)."""
        reg = weights.c_reg()
        lay = _clayout(layout)
        vals = np.zeros(4)
        g = None if device_only else (np.zeros(layout["total"]) if grad is None else grad)
        self._chk(self.L.cdr_regularisers(self.h, C.byref(reg), C.byref(lay), _dp(vals), _dp(g)))
        return dict(zip(("normal", "edge", "spec", "roug"), vals.tolist())), g

    def grad_image_loss(self, view, target, settings: RenderSettings, lambda_rend, use_target_mask, layout,
                        grad=None, target_mask=None):
        """grad_image_loss (diff_render.cpp:285-305): one view, no Laplacian."""
        self.set_target(view, target, target_mask)
        loss, g, _, _ = self.loss_grad([view], settings, layout, lambda_rend, 0.0, 0, use_target_mask, grad=grad)
        return loss[0], g

    def cotangent_laplacian(self, mode=0):
        nnz = C.c_int64()
        self._chk(self.L.cdr_laplacian_matrix(self.h, mode, None, None, None, C.byref(nnz)))
        outer = np.zeros(self.V + 1, np.int32)
        inner = np.zeros(nnz.value, np.int32)
        vals = np.zeros(nnz.value)
        self._chk(self.L.cdr_laplacian_matrix(self.h, mode, _ip(outer), _ip(inner), _dp(vals), C.byref(nnz)))
        return outer, inner, vals

    def laplacian_loss(self, mode=0, lam=0.1):
        g = np.zeros((self.V, 3))
        v = C.c_double()
        self._chk(self.L.cdr_laplacian_loss(self.h, mode, lam, C.byref(v), _dp(g)))
        return v.value, g

    # ---- resident optimiser: total_loss -> adam -> evolve
    def adam_init(self, config: AdamConfig, layout):
        """AdamState(layout, config) on the device (m = v = 0, step 0)."""
        self._adam_layout = layout
        self._chk(self.L.cdr_adam_init(self.h, C.byref(config.c()), C.byref(_clayout(layout))))

    def adam_step(self, want_displacement=True):
        """adam_step + apply on the resident parameters with the device gradient
        of the last loss pass. Returns (displacement V x 3 or None, step)."""
        disp = np.zeros((self.V, 3)) if want_displacement else None
        step = C.c_int64()
        self._chk(self.L.cdr_adam_step(self.h, _dp(disp), C.byref(step)))
        return disp, step.value

    def adam_state(self):
        n = self._adam_layout["total"]
        m, v, step = np.zeros(n), np.zeros(n), C.c_int64()
        self._chk(self.L.cdr_adam_get_state(self.h, _dp(m), _dp(v), C.byref(step)))
        return m, v, step.value

    def set_adam_state(self, m, v, step):
        self._chk(self.L.cdr_adam_set_state(self.h, _dp(np.ascontiguousarray(m, dtype=np.float64)),
                                            _dp(np.ascontiguousarray(v, dtype=np.float64)), int(step)))

    def evolve(self, displacement=None, want_positions=True):
        """robust_evolve on the device (the displacement of the last adam_step
        when None). Returns (applied scale, positions V x 3 or None)."""
        d = None if displacement is None else np.ascontiguousarray(displacement, dtype=np.float64)
        out = np.zeros((self.V, 3)) if want_positions else None
        sc = C.c_double()
        self._chk(self.L.cdr_evolve(self.h, _dp(d), C.byref(sc), _dp(out)))
        return sc.value, out

    def params(self, layout):
        """pack (params.cpp:70-100) of the resident state."""
        out = np.zeros(layout["total"])
        self._chk(self.L.cdr_get_params(self.h, C.byref(_clayout(layout)), _dp(out)))
        return out

    def lbvh_keys(self):
        """Sorted LBVH leaf keys (Morton << 32 | face) of the current mesh."""
        n = self.T
        out = np.zeros(n, np.uint64)
        self._chk(self.L.cdr_lbvh_keys(self.h, out.ctypes.data_as(C.POINTER(C.c_uint64)), n))
        return out

    def rendered(self, view):
        """(rgb H x W x 3, mask H x W) of the last pass that rendered `view`."""
        cam = self.cameras[view]
        rgb = np.zeros((cam.height, cam.width, 3))
        mask = np.zeros((cam.height, cam.width))
        self._chk(self.L.cdr_get_rendered(self.h, view, _dp(rgb), _dp(mask)))
        return rgb, mask

    def closest_points(self, positions, triangles, queries):
        """Bvh::closest_point (bvh.cpp:267-329) of each query on any mesh:
        (tri, point n x 3, distance, barycentrics n x 3)."""
        pos = np.ascontiguousarray(positions, dtype=np.float64)
        tris = np.ascontiguousarray(triangles, dtype=np.int32)
        q = np.ascontiguousarray(queries, dtype=np.float64)
        n = len(q)
        tri, pt, di, ba = np.zeros(n, np.int32), np.zeros((n, 3)), np.zeros(n), np.zeros((n, 3))
        self._chk(self.L.cdr_closest_points(self.h, _dp(pos), len(pos), _ip(tris), len(tris), _dp(q), n, _ip(tri),
                                            _dp(pt), _dp(di), _dp(ba)))
        return tri, pt, di, ba

    def point_to_mesh_distance(self, points, positions, triangles):
        """point_to_mesh_distance (mesh.cpp:127-133): mean closest distance."""
        if len(triangles) == 0:
            raise CollodiffError("mesh has no triangles")  # EmptyMesh
        _, _, d, _ = self.closest_points(positions, triangles, points)
        s = 0.0
        for x in d:  # the reference's sequential sum
            s += float(x)
        return s / len(d) if len(d) else 0.0

    def uv_transfer(self, old_positions, old_triangles, old_uvs, new_positions, max_distance):
        """uv_transfer (remesh.cpp:281-294): UVs of new vertices from the
        closest point on the old mesh; ProjectionTooFar past max_distance."""
        tri, _, d, b = self.closest_points(old_positions, old_triangles, new_positions)
        bad = np.nonzero((tri < 0) | (d > max_distance))[0]
        if len(bad):
            v = int(bad[0])
            raise ProjectionTooFar(f"uv transfer: vertex {v} is {d[v]} away from the source mesh")
        t = np.asarray(old_triangles)[tri]
        uv = np.asarray(old_uvs, dtype=np.float64)
        return (uv[t[:, 0]] * b[:, :1] + uv[t[:, 1]] * b[:, 1:2]) + uv[t[:, 2]] * b[:, 2:3]

    def self_intersects(self, positions, triangles, want_pairs=False):
        """self_intersects (mesh.hpp:67) of any mesh (not necessarily this
        renderer's): (bool, pairs (n x 2, sorted by (f, g)) or None)."""
        pos = np.ascontiguousarray(positions, dtype=np.float64)
        tris = np.ascontiguousarray(triangles, dtype=np.int32)
        res = C.c_int32()
        if not want_pairs:
            self._chk(self.L.cdr_self_intersects(self.h, _dp(pos), len(pos), _ip(tris), len(tris), C.byref(res),
                                                 None, 0, None))
            return bool(res.value), None
        n = C.c_int64()
        cap = max(16, 4 * len(tris))
        pairs = np.zeros((cap, 2), np.int32)
        self._chk(self.L.cdr_self_intersects(self.h, _dp(pos), len(pos), _ip(tris), len(tris), C.byref(res),
                                             _ip(pairs), cap, C.byref(n)))
        if n.value > cap:
            pairs = np.zeros((n.value, 2), np.int32)
            self._chk(self.L.cdr_self_intersects(self.h, _dp(pos), len(pos), _ip(tris), len(tris), C.byref(res),
                                                 _ip(pairs), n.value, C.byref(n)))
        return bool(res.value), pairs[:n.value].copy()

    def grad_device(self):
        p = _vp()
        n = C.c_int64()
        self._chk(self.L.cdr_grad_device_ptr(self.h, C.byref(p), C.byref(n)))
        return p.value, n.value

    def get_grad(self, n):
        out = np.zeros(n)
        self._chk(self.L.cdr_get_grad(self.h, _dp(out), n))
        return out

    def set_grad(self, g):
        g = np.ascontiguousarray(g, dtype=np.float64)
        self._chk(self.L.cdr_set_grad(self.h, _dp(g), len(g)))

    # ---------------------------------------------------------------- multi-GPU
    @staticmethod
    def nccl_unique_id() -> bytes:
        L = load_library()
        buf = C.create_string_buffer(128)
        rc = L.cdr_nccl_unique_id(buf)
        if rc != 0:
            raise CollodiffError("ncclGetUniqueId failed (NCCL not loadable?)")
        return buf.raw

    def comm_init(self, uid: bytes, n_ranks: int, rank: int):
        self._chk(self.L.cdr_comm_init(self.h, C.c_char_p(uid), n_ranks, rank))

    def set_rank(self, rank: int, n_ranks: int):
        """Shard of a group summed by the caller (no communicator): only rank 0
        adds the Laplacian and the regularisers."""
        self._chk(self.L.cdr_set_rank(self.h, rank, n_ranks))

    @staticmethod
    def comm_init_all(renderers):
        """One process, one context per device: ncclCommInitAll over them."""
        L = load_library()
        arr = (_vp * len(renderers))(*[r.h for r in renderers])
        rc = L.cdr_comm_init_all(arr, len(renderers))
        if rc != 0:
            raise _ERRORS.get(rc, CollodiffError)(L.cdr_last_error(renderers[0].h).decode())

    def comm_info(self):
        """(ranks, rank) as NCCL's communicator reports them (ncclCommCount /
        ncclCommUserRank); (1, 0) without a communicator."""
        n, r = C.c_int32(), C.c_int32()
        self._chk(self.L.cdr_comm_info(self.h, C.byref(n), C.byref(r)))
        return n.value, r.value


def device_count() -> int:
    L = load_library()
    n = C.c_int()
    L.cdr_device_count(C.byref(n))
    return n.value


__all__ = ["Renderer", "RenderSettings", "param_layout", "SizeMismatch", "NonFiniteGradient", "CollodiffError",
           "load_library", "SEGMENT_DTYPE", "CAMERA_DTYPE", "device_count"]
