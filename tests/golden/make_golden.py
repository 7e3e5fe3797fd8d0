"""Generate tests/golden/*.npz from the REFERENCE library compiled from its own
sources (oracle/_ref). Run where /root/reference exists:

    python tests/golden/make_golden.py

Each fixture stores the inputs (so it is self-contained) and the reference's
outputs: hit caches, images, masks, per-view loss + adjoint, interior and
boundary gradients, silhouette segments, the Laplacian (CSC, value, gradient)
the hot subset of total_loss (loss terms + gradient), the four mesh/material
regularisers at two weight sets (REG_WEIGHTS) and total_loss with every term
at the reference default weights (LossWeights, losses.hpp:14-23); and
selfint.npz: self_intersects pairs of clean, broken and noisy meshes;
optimize.npz: adam_step and robust_evolve cases; closest.npz:
Bvh::closest_point, point_to_mesh_distance and uv_transfer cases.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.pyoracle import (RefLib, adam_step, closest_points, layout_for, ref_point_to_mesh,  # noqa: E402
                             ref_self_intersects, ref_uv_transfer, robust_evolve)
from paper_2103_15208_b200 import scenes as S  # noqa: E402

# (normal, edge, spec, roug, sigma1, sigma2): the reference defaults, then a
# second set with other sigmas so the window weights are exercised off-default
REG_WEIGHTS = {"default": (0.01, 1.0, 0.01, 0.001, 2.0, 0.1), "alt": (0.3, 0.7, 0.05, 0.02, 1.3, 0.25)}

CASES = {
    "sphere_f4": dict(mesh=lambda: S.geodesic_sphere(4), tex=8, views=2, image=24, spp=4, seed=3, light=True),
    "blob_f5": dict(mesh=lambda: S.blob(5), tex=16, views=2, image=32, spp=9, seed=1, light=False),
}


def make(name, c):
    sc = S.make_scene(c["mesh"](), c["tex"], c["views"], c["image"])
    ts = S.perturbed_target_scene(sc)
    ref, tref = RefLib(sc), RefLib(ts)
    spp, seed = c["spp"], c["seed"]
    lay = layout_for(sc, optimize_light=c["light"])
    out = dict(positions=sc.mesh.positions, triangles=sc.mesh.triangles, uvs=sc.mesh.uvs, edges=sc.mesh.edges,
               diffuse=sc.diffuse, specular=sc.specular, roughness=sc.roughness, light=sc.light,
               background=sc.background, cameras=S.camera_struct_array(sc.cameras), spp=spp, seed=seed,
               optimize_light=int(c["light"]))
    targets = np.stack([tref.render(v, spp, seed + 0x7A9)[0] for v in range(c["views"])])
    out["targets"] = targets
    for v in range(c["views"]):
        rgb, mask, hit = ref.render(v, spp, seed)
        val, adj = ref.view_loss(rgb, targets[v])
        out[f"v{v}_rgb"], out[f"v{v}_mask"], out[f"v{v}_hit"] = rgb, mask, hit
        out[f"v{v}_loss"], out[f"v{v}_adj"] = np.array(val), adj
        out[f"v{v}_interior"] = ref.interior(v, adj, spp, seed, hit, lay)
        segs, tot = ref.silhouettes(v)
        out[f"v{v}_segments"], out[f"v{v}_seglen"] = segs, np.array(tot)
        g, deg = ref.boundary(v, adj, c["image"] ** 2, seed, lay)
        out[f"v{v}_boundary"], out[f"v{v}_degenerate"] = g, np.array(deg)
    val, grad, (o_, i_, x_) = ref.laplacian(0, 0.1)
    out.update(lap_value=np.array(val), lap_grad=grad, lap_outer=o_, lap_inner=i_, lap_vals=x_)
    bd, g, _ = ref.total_loss(targets, spp, seed, lay)
    out["total_breakdown"], out["total_grad"] = bd, g
    for k, w in REG_WEIGHTS.items():
        vals, gp, gd, gs, gr = ref.regularisers(w)
        out.update({f"reg_{k}_values": vals, f"reg_{k}_pos": gp, f"reg_{k}_diffuse": gd, f"reg_{k}_specular": gs,
                    f"reg_{k}_roughness": gr, f"reg_{k}_w": np.array(w)})
    bd, g, _ = ref.total_loss(targets, spp, seed, lay, others=REG_WEIGHTS["default"][:4])
    out["full_breakdown"], out["full_grad"] = bd, g
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print(name, os.path.getsize(os.path.join(HERE, name + ".npz")), "bytes")


def selfint_cases():
    """Meshes for self_intersects (mesh.cpp:184-214): clean, broken and noisy."""
    rng = np.random.default_rng(11)
    out = {}
    ico = S.icosphere(2)
    out["ico2"] = (ico.positions, ico.triangles)
    p = ico.positions.copy()
    p[0] = -p[0] * 1.2  # test_mesh.cpp:126-131
    out["ico2_punched"] = (p, ico.triangles)
    out["two_tris"] = (np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0.3, 0.3, -1], [0.5, 0.1, 1], [0.1, 0.5, 1.0]]),
                       np.array([[0, 1, 2], [3, 4, 5]], np.int32))  # test_mesh.cpp:116-124
    for name, m in (("sphere_f12", S.geodesic_sphere(12)), ("knot_small", S.torus_knot(120, 10))):
        out[name] = (m.positions, m.triangles)
        scale = np.ptp(m.positions, axis=0).max()
        for k, sd in enumerate((0.002, 0.01, 0.04)):
            out[f"{name}_noise{k}"] = (m.positions + rng.normal(0, sd * scale, m.positions.shape), m.triangles)
    return out


def make_selfint():
    out = {}
    for name, (pos, tris) in selfint_cases().items():
        b, pairs = ref_self_intersects(pos, tris)
        out[f"{name}_pos"], out[f"{name}_tris"] = np.asarray(pos, np.float64), np.asarray(tris, np.int32)
        out[f"{name}_result"], out[f"{name}_pairs"] = np.array(int(b)), pairs
        print(name, len(tris), "tris", int(b), len(pairs), "pairs")
    np.savez_compressed(os.path.join(HERE, "selfint.npz"), names=np.array(sorted(selfint_cases())), **out)


ADAM_CFG = (0.9, 0.999, 1e-8, 2e-3, 1e-2, 5e-2)


def make_optimize():
    """adam_step (adam.cpp:9-54) and robust_evolve (evolve.cpp:19-53) cases."""
    rng = np.random.default_rng(21)
    out = {"adam_cfg": np.array(ADAM_CFG)}
    sc = S.make_scene(S.icosphere(2), 8, 1, 16)
    for light in (0, 1):
        lay = layout_for(sc, optimize_light=bool(light))
        n, V = lay["total"], sc.mesh.V
        params = rng.uniform(-0.05, 1.05, n)  # some outside [0, 1]: the clamps
        grad = rng.normal(0, 1, n)
        grad[rng.uniform(size=n) < 0.2] = 0.0
        m, v = rng.normal(0, 0.1, n), rng.uniform(0, 0.1, n)
        for step in (0, 6):
            rc, st, m2, v2, p2, d2 = adam_step(ADAM_CFG, lay, V, (8, 8), step, m, v, params, grad, ref=True)
            k = f"adam_l{light}_s{step}"
            out.update({f"{k}_params": params, f"{k}_grad": grad, f"{k}_m": m, f"{k}_v": v, f"{k}_m2": m2,
                        f"{k}_v2": v2, f"{k}_p2": p2, f"{k}_d2": d2, f"{k}_step2": np.array(st)})
    m = S.blob(4)
    out["evolve_pos"], out["evolve_tris"] = m.positions, m.triangles
    for k, sd in enumerate((0.0, 0.002, 0.02, 0.08, 0.5, 3.0, 40.0)):
        d = rng.normal(0, sd, m.positions.shape)
        rc, pos, scale = robust_evolve(m.positions, m.triangles, d, ref=True)
        out.update({f"evolve{k}_d": d, f"evolve{k}_pos": pos, f"evolve{k}_scale": np.array(scale),
                    f"evolve{k}_rc": np.array(rc)})
        print("evolve", k, sd, rc, scale)
    p = S.icosphere(2)
    bad = p.positions.copy()
    bad[0] = -bad[0] * 1.2
    rc, _, _ = robust_evolve(bad, p.triangles, np.zeros_like(bad), ref=True)
    out.update({"evolve_bad_pos": bad, "evolve_bad_tris": p.triangles, "evolve_bad_rc": np.array(rc)})
    print("evolve bad input", rc)
    np.savez_compressed(os.path.join(HERE, "optimize.npz"), **out)


def make_closest():
    """Bvh::closest_point, point_to_mesh_distance and uv_transfer cases."""
    rng = np.random.default_rng(41)
    m = S.blob(6)
    q = np.concatenate([rng.normal(0, 0.6, (1500, 3)),              # volume: many edge/vertex ties
                        m.positions[:300] * 1.0001,                  # just off vertices
                        m.positions[rng.integers(0, m.V, 200)] + rng.normal(0, 1e-3, (200, 3))])
    tri, pt, di, ba = closest_points(m.positions, m.triangles, q, ref=True)
    out = {"pos": m.positions, "tris": m.triangles, "uvs": m.uvs, "q": q, "tri": tri, "pt": pt, "dist": di,
           "bary": ba, "p2m": np.array(ref_point_to_mesh(m.positions, m.triangles, q))}
    fine = S.blob(9)  # a finer sampling of the same surface: a remesh's new vertices
    rc, uv = ref_uv_transfer(m.positions, m.triangles, m.uvs, fine.positions, 0.05)
    out.update({"new_pos": fine.positions, "uv_rc": np.array(rc), "uv": uv})
    rc2, _ = ref_uv_transfer(m.positions, m.triangles, m.uvs, fine.positions * 1.5, 0.05)
    out["uv_far_rc"] = np.array(rc2)
    print("closest", len(q), "queries; uv_transfer", rc, "far", rc2)
    np.savez_compressed(os.path.join(HERE, "closest.npz"), **out)


if __name__ == "__main__":
    for n, c in CASES.items():
        make(n, c)
    make_selfint()
    make_optimize()
    make_closest()
