"""Uniform test adapter over the two implementations of the hot path:
the CPU oracle (oracle/cdr_oracle.c) and the GPU product (libcdr.so)."""
import numpy as np

from oracle.pyoracle import Oracle
from paper_2103_15208_b200.api import RenderSettings, Renderer


class OracleBackend:
    name = "oracle"

    def __init__(self, scene, view_ids=None):
        self.o = Oracle(scene, view_ids)
        self.scene = scene

    def render(self, v, spp, seed):
        return self.o.render(v, spp, seed)

    def radiance_at(self, v, xy):
        return self.o.radiance_at(v, np.asarray(xy, dtype=np.float64).reshape(-1, 2))

    def silhouettes(self, v):
        return self.o.silhouettes(v)

    def laplacian(self, mode, lam=0.1):
        v, g, (outer, inner, vals) = self.o.laplacian(mode, lam)
        return outer, inner, vals

    def lv(self, mode):
        outer, inner, vals = self.laplacian(mode)
        return csc_times(outer, inner, vals, self.scene.mesh.positions)


class GpuBackend(OracleBackend):
    name = "gpu"

    def __init__(self, scene, view_ids=None):
        self.r = Renderer(0, scene, view_ids)
        self.scene = scene

    def render(self, v, spp, seed):
        return self.r.render(v, RenderSettings(spp=spp, seed=seed))

    def radiance_at(self, v, xy):
        return self.r.radiance_at(v, np.asarray(xy, dtype=np.float64).reshape(-1, 2))

    def silhouettes(self, v):
        return self.r.extract_silhouettes(v)

    def laplacian(self, mode, lam=0.1):
        return self.r.cotangent_laplacian(mode)


def csc_times(outer, inner, vals, x):
    out = np.zeros((len(outer) - 1, x.shape[1]))
    for j in range(len(outer) - 1):
        for k in range(outer[j], outer[j + 1]):
            out[inner[k]] += vals[k] * x[j]
    return out


def make(kind, scene, view_ids=None):
    return (GpuBackend if kind == "gpu" else OracleBackend)(scene, view_ids)
