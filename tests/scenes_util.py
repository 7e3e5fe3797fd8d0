"""Shared small test scenes (fed identically to the GPU path and the oracles)."""
import numpy as np

from paper_2103_15208_b200 import scenes as S


def small_scene(freq=4, tex=16, views=2, image=32, seed=7):
    return S.make_scene(S.geodesic_sphere(freq), tex, views, image, seed=seed)


def blob_scene(freq=8, tex=32, views=2, image=48):
    return S.make_scene(S.blob(freq), tex, views, image)


def targets_for(scene, spp, seed, oracle_cls):
    """Targets rendered from the perturbed scene (gradcheck.cpp:49-73)."""
    ts = S.perturbed_target_scene(scene)
    o = oracle_cls(ts)
    return np.stack([o.render(v, spp, seed + 0x7A9)[0] for v in range(len(scene.cameras))])


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)
