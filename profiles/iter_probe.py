import sys, time, os
sys.path.insert(0, "/root/repo")
import numpy as np
import bench
from paper_2103_15208_b200 import api, scenes as S
scene, gids, cfg, total = bench.build_workload("cfg2", 0, 1, None)
r = api.Renderer(0, scene, view_ids=gids)
tr = api.Renderer(0, S.perturbed_target_scene(scene), view_ids=gids)
for k in range(len(scene.cameras)):
    img, _, _ = tr.render(k, api.RenderSettings(spp=16, seed=1 + 0x7A9), want_hits=False)
    r.set_target(k, img)
tr.close()
lay = api.param_layout(scene)
st = api.RenderSettings(spp=16, seed=1)
views = np.arange(len(scene.cameras), dtype=np.int32)
lw = api.LossWeights()
diag = float(np.linalg.norm(np.ptp(scene.mesh.positions, axis=0)))
r.adam_init(api.AdamConfig(lr_positions=1e-3 * diag), lay)
def timeit(name, fn, n=5):
    fn()
    out = []
    for _ in range(n):
        t0 = time.perf_counter(); s = fn(); out.append((1e3 * (time.perf_counter() - t0), s))
    print(name, [round(x[0], 2) for x in out], [round(x[1].ms_total, 2) if x[1] is not None else None for x in out])
timeit("loss_grad", lambda: r.loss_grad(views, st, lay, device_only=True)[2])
timeit("total_loss_device", lambda: r.total_loss_device(views, st, lay, lw)[1])
def it():
    _, s = r.total_loss_device(views, st, lay, lw); r.adam_step(want_displacement=False); r.evolve(want_positions=False); return s
timeit("iteration", it)
timeit("loss_grad after", lambda: r.loss_grad(views, st, lay, device_only=True)[2])
# the bench's iteration loop (2 warm + 20 timed), per-iteration wall and device ms
rows = []
for i in range(22):
    t0 = time.perf_counter()
    bd, s = r.total_loss_device(views, st, lay, lw)
    t1 = time.perf_counter()
    r.adam_step(want_displacement=False)
    sc, _ = r.evolve(want_positions=False)
    rows.append((round(1e3 * (t1 - t0), 1), round(s.ms_total, 1), round(s.ms_render, 1), round(s.ms_trace, 1), round(s.ms_boundary, 1), s.segments, s.hit_samples, s.beam_fallback_tiles, s.shaded_samples, round(bd["total"], 2), sc))
for row in rows:
    print(row)
