"""Probe-path statistics of the boundary pass at a bench config (debug build
with -DCDR_TRACE_STATS): which path each probe takes, scan steps, per-ray
traversal cost."""
import ctypes as C, json, os, sys
sys.path.insert(0, "/root/repo")
os.environ["CDR_LIB"] = sys.argv[2]
import numpy as np
import bench
from paper_2103_15208_b200 import api, scenes as S
cfgname = sys.argv[1]
scene, gids, cfg, total = bench.build_workload(cfgname, 0, 1, None)
r = api.Renderer(0, scene, view_ids=gids)
tr = api.Renderer(0, S.perturbed_target_scene(scene), view_ids=gids)
for k in range(len(scene.cameras)):
    img, _, _ = tr.render(k, api.RenderSettings(spp=cfg["spp"], seed=1 + 0x7A9), want_hits=False)
    r.set_target(k, img)
tr.close()
lay = api.param_layout(scene)
st = api.RenderSettings(spp=cfg["spp"], seed=1)
views = np.arange(len(scene.cameras), dtype=np.int32)
L = api.load_library()
buf8 = (C.c_ulonglong * 8)(); buf4 = (C.c_ulonglong * 4)()
r.loss_grad(views, st, lay, device_only=True)
L.cdr_debug_probe_stats(buf8); L.cdr_debug_trace_stats_boundary(buf4); L.cdr_debug_trace_stats(buf4)
_, _, s, _ = r.loss_grad(views, st, lay, device_only=True)
L.cdr_debug_probe_stats(buf8)
L.cdr_debug_trace_stats_boundary(buf4)
names = ["per_ray_offimage", "per_ray_overflow", "small_list", "big_list", "small_tile_scan", "big_tile_scan",
         "scan_steps", "empty_list"]
ps = dict(zip(names, list(buf8)))
n = sum(v for k, v in ps.items() if k != "scan_steps")
ts = list(buf4)
print(json.dumps({"config": cfgname, "probes": n, "paths": {k: v / n for k, v in ps.items() if k != "scan_steps"},
                  "scan_steps_per_listed_probe": ps["scan_steps"] / max(1, n - ps["per_ray_offimage"] - ps["per_ray_overflow"]),
                  "per_ray": {"rays": ts[0], "node_visits_per_ray": ts[1] / max(1, ts[0]), "leaf_tests_per_ray": ts[2] / max(1, ts[0])},
                  "ms_boundary": s.ms_boundary, "fallback_tiles": s.beam_fallback_tiles}, indent=1))
