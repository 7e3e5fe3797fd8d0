"""One optimisation iteration of a bench config, bracketed for ncu
(--profile-from-start off): every kernel the library launches in
total_loss (all six terms) -> adam_step -> robust_evolve, after one warm-up
iteration, with the targets already rendered (outside the bracket).

    ncu --profile-from-start off --set full ... python profiles/profile_step.py --config cfg4
    ncu --profile-from-start off --metrics gpu__time_duration.sum ... python profiles/profile_step.py ...

The launch list of the same bracket gives each kernel's share of the step.
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--views", type=int, default=None)
    ap.add_argument("--loss-only", action="store_true", help="bracket only the loss call")
    ap.add_argument("--bench-step", action="store_true",
                    help="bracket bench.py's timed step instead: cdr_loss_grad over the synthetic maps "
                         "(fp32 texel records), no regularisers, no optimiser step")
    a = ap.parse_args()
    import torch
    import bench
    from paper_2103_15208_b200 import api
    from paper_2103_15208_b200 import scenes as S
    scene, gids, cfg, total = bench.build_workload(a.config, 0, 1, a.views)
    spp, seed = cfg["spp"], 1
    r = api.Renderer(0, scene, view_ids=gids)
    tr = api.Renderer(0, S.perturbed_target_scene(scene), view_ids=gids)
    for k in range(len(scene.cameras)):
        img, _, _ = tr.render(k, api.RenderSettings(spp=spp, seed=seed + 0x7A9), want_hits=False)
        r.set_target(k, img)
    tr.close()
    lay = api.param_layout(scene)
    st = api.RenderSettings(spp=spp, seed=seed)
    views = np.arange(len(scene.cameras), dtype=np.int32)
    diag = float(np.linalg.norm(np.ptp(scene.mesh.positions, axis=0)))
    r.adam_init(api.AdamConfig(lr_positions=1e-3 * diag), lay)
    lw = api.LossWeights()

    if a.bench_step:
        r.loss_grad(views, st, lay, device_only=True)  # warm-up
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        _, _, stats, _ = r.loss_grad(views, st, lay, device_only=True)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        print({"config": a.config, "views": len(views), "bench_step": True, "launches": stats.kernel_launches})
        r.close()
        return

    def iteration():
        bd, stats = r.total_loss_device(views, st, lay, lw)
        if not a.loss_only:
            r.adam_step(want_displacement=False)
            r.evolve(want_positions=False)
        return bd, stats

    iteration()  # warm-up (module load, pool sizing)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    bd, stats = iteration()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print({"config": a.config, "views": len(views), "loss": bd["total"], "launches": stats.kernel_launches,
           "ms_total": stats.ms_total})
    r.close()


if __name__ == "__main__":
    main()
