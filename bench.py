#!/usr/bin/env python
"""Benchmark of the B200 differentiable-rendering hot path (one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg1..cfg5] [--views K]

--gpus N > 1 without torchrun's environment re-executes this script under
`torch.distributed.run --nproc-per-node N` (one rank per GPU; exits non-zero
when fewer than N devices exist). Under torchrun every rank drives one GPU:
the config's views are sharded by global view id and the gradient is summed
by the library's NCCL all-reduce inside cdr_loss_grad. The default config is
cfg2 (BASELINE configs[1]: 50 views, weak scaling) at N = 1 and cfg3
(configs[2]: 100 views split over the ranks, strong scaling) at N > 1.

A step = the hot subset of total_loss (losses.cpp:244-297) over the rank's
views: per-iteration LBVH rebuild + normals, fused trace/shade/loss/interior,
silhouettes + boundary edge sampling, normal chain, cotangent Laplacian.
  value : device-timed (CUDA events on the library's stream, L2 flushed
          before each step), inputs resident in HBM, gradient left on device.
  e2e   : the same step through the C-ABI with HOST buffers: positions and the
          three texture maps uploaded from pinned memory and the gradient
          downloaded every step (wall clock around the blocking C-ABI calls:
          cdr_stage_params + cdr_loss_grad, which overlaps the copies with its
          kernels; e2e.separate_uploads = synchronous uploads before the call;
          no L2 flush between e2e steps, so with the copies hidden e2e can
          exceed the L2-flushed device value);
          e2e.with_rendered_images adds total_loss's K rendered images + masks
          (TotalLossResult::rendered, losses.cpp:259) to the download.
  cpu_baseline : the reference library compiled from its own sources
          (oracle/_ref; the C oracle port if absent) on the fixed 4-view subset
          of BASELINE.md §3.4 (global views 0-3), all host threads, rank 0 at
          N = 1 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fwd+adjoint Msamples/s at 1/2/4/8 B200; ms per optimisation iteration"
UNIT = "Msamples/s"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0}
# BASELINE.json configs (SURVEY.md §8(d) shapes). cfg2 (configs[1]) is the
# default and the driver's line; the others are reachable with --config.
# weak: every rank owns `views` views; strong: `views` views split over ranks.
CONFIGS = {
    "cfg1": dict(mesh="geodesic_sphere(11): 2,420 tris", tex=128, views=4, image=128, spp=4, scaling="weak"),
    "cfg2": dict(mesh="blob(59): 69,620 tris", tex=512, views=50, image=512, spp=16, scaling="weak"),
    "cfg3": dict(mesh="blob(59): 69,620 tris", tex=1024, views=100, image=512, spp=16, scaling="strong"),
    "cfg4": dict(mesh="torus_knot(1000x100): 200,000 tris", tex=1024, views=64, image=1024, spp=16,
                 scaling="strong"),
    "cfg5": dict(mesh="blob(59): 69,620 tris", tex=1024, views=400, image=512, spp=16, scaling="strong"),
}


def workload_text(name, cfg, views):
    return (f"{name}: {cfg['mesh']}, {cfg['tex']}^2 SVBRDF textures, {views} views at {cfg['image']}^2, "
            f"{cfg['spp']} spp, boundary term M=W*H, cotangent Laplacian ({cfg['scaling']} scaling)")


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def parse(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default=None, choices=sorted(CONFIGS),
                   help="default: cfg2 at one GPU, cfg3 (strong scaling) at N > 1")
    p.add_argument("--views", type=int, default=None, help="override the config's view count")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-iteration", action="store_true", help="skip the resident optimisation-iteration timing")
    return p.parse_args(argv)


def build_workload(name, rank, world, n_views=None):
    from paper_2103_15208_b200 import scenes as S
    from paper_2103_15208_b200.shard import shard_views, weak_views
    cfg = CONFIGS[name]
    mesh = {"cfg1": lambda: S.geodesic_sphere(11), "cfg4": lambda: S.torus_knot()}.get(name, lambda: S.blob(59))()
    d, s, r = S.random_maps(cfg["tex"], seed=7)
    views = n_views or cfg["views"]
    if cfg["scaling"] == "weak":
        total, gids = views * world, weak_views(views, rank)
    else:
        total, gids = views, shard_views(views, world, rank)
    cams = S.sample_views_on_sphere(total, 2.5, 11, 40.0, cfg["image"], cfg["image"])
    scene = S.Scene(mesh, d, s, r, [cams[g] for g in gids])
    return scene, gids, cfg, total


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return PEAKS_FALLBACK, "fallback"


class NvmlClockSampler:
    """SM clock and clock-event reasons during the timed region, polled through
    NVML from a thread every 5 ms (a timed region of ~100 ms is shorter than an
    nvidia-smi process takes to start, so that sampler sees one row at best)."""

    def __init__(self, device):
        import threading
        import pynvml as nv
        nv.nvmlInit()
        self.nv = nv
        self.h = nv.nvmlDeviceGetHandleByIndex(device)
        self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
        self.rows = []
        self.halt = threading.Event()
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def _run(self):
        nv = self.nv
        while not self.halt.is_set():
            try:
                self.rows.append((nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM),
                                  nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)))
            except Exception:
                pass
            self.halt.wait(0.005)

    def stop(self):
        self.halt.set()
        self.t.join(timeout=5)
        nv = self.nv
        bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["no samples"], "source": "nvml"}
        sm = [r[0] for r in self.rows]
        loaded = [x for x in sm if x > 0.5 * self.max_mhz] or sm
        reasons = sorted({n for _, m in self.rows for n, b in bits.items() if m & b})
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.rows), "source": "nvml, 5 ms"}


def clock_sampler(device):
    try:
        return NvmlClockSampler(device)
    except Exception:
        return ClockSampler(device)


class ClockSampler:
    """nvidia-smi clocks/throttle reasons during the timed region."""

    def __init__(self, device):
        self.f = tempfile.NamedTemporaryFile(mode="w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(device), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        rows = []
        with open(self.f.name) as fh:
            for line in fh:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [num(r[1]) for r in rows if num(r[1]) is not None]
        mx = [num(r[2]) for r in rows if num(r[2]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        loaded = [x for x in sm if mx and x > 0.5 * max(mx)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


CPU_SUBSET = 4  # a fixed 4-view subset (global views 0-3)


def cpu_baseline_sample(scene, spp, seed, lay, threads, kind_pref="reference", label="cfg2", views=None):
    """Reference total_loss on a bounded sample: the given camera indices of
    `scene` (default the first CPU_SUBSET), one total_loss call each."""
    from oracle import pyoracle
    from paper_2103_15208_b200 import scenes as S
    views = list(range(min(CPU_SUBSET, len(scene.cameras)))) if views is None else list(views)
    kind = "reference" if kind_pref == "reference" else "port"
    dt, samples = 0.0, 0
    for v in views:
        one = S.Scene(scene.mesh, scene.diffuse, scene.specular, scene.roughness, [scene.cameras[v]])
        tscene = S.perturbed_target_scene(one)
        try:
            if kind != "reference":
                raise FileNotFoundError
            ref = pyoracle.RefLib(one)
            tgt = pyoracle.RefLib(tscene).render(0, spp, seed + 0x7A9, threads=threads)[0][None]

            def run():
                return ref.total_loss(tgt, spp, seed, lay, threads=threads)
        except (FileNotFoundError, OSError):
            kind, threads = "port", 1
            orc = pyoracle.Oracle(one)
            tgt = pyoracle.Oracle(tscene).render(0, spp, seed + 0x7A9)[0][None]
            st = pyoracle.settings(spp, seed)

            def run():
                return orc.loss_grad(tgt, st, lay)
        t0 = time.perf_counter()
        run()
        dt += time.perf_counter() - t0
        cam = one.cameras[0]
        samples += cam.width * cam.height * spp
    cam = scene.cameras[views[0]]
    return {"value": samples / dt / 1e6, "unit": UNIT, "cores": threads, "kind": kind,
            "sample": f"{len(views)} {label} view(s) (cameras {views}; {cam.width}^2 x {spp} spp, "
                      f"{scene.mesh.T:,} tris, {scene.tex_res[0]}^2 tex), one total_loss each, {dt:.2f} s wall",
            "seconds": dt, "samples": samples}


def run_reference(args, rank, world):
    """The reference arm: oracle/_ref (the reference compiled from its own
    sources) on the host cores; each step = total_loss of one view of the
    4-view subset, cycling through it. Rank 0 only."""
    if rank != 0:
        return 0
    from paper_2103_15208_b200 import api
    name = args.config
    scene, gids, cfg, total = build_workload(name, 0, 1)  # the config's camera set; views 0-3 are sampled
    lay = api.param_layout(scene)
    threads = os.cpu_count() or 1
    secs, samples = [], 0
    cb = None
    for i in range(args.warmup + args.steps):
        cb = cpu_baseline_sample(scene, cfg["spp"], 1, lay, threads, label=name,
                                 views=[i % min(CPU_SUBSET, len(scene.cameras))])
        if i >= args.warmup:
            secs.append(cb["seconds"])
            samples += cb["samples"]
    dt = sum(secs)
    v = samples / dt / 1e6
    line = {"metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * dt / len(secs), "higher_is_better": True,
            "scaling": cfg["scaling"], "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_text(name, cfg, CONFIGS[name]["views"]), "name": name,
                       "sample": f"1 view per step, cycling through the {CPU_SUBSET}-view subset (global views "
                                 f"0-{CPU_SUBSET - 1}, BASELINE.md §3.4) (bounded CPU sample)",
                       "threads": threads},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cb["cores"], "kind": cb["kind"],
                             "sample": f"{len(secs)} steps x 1 view of the {CPU_SUBSET}-view subset through "
                                       f"total_loss, {dt:.2f} s wall"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def launch_command(argv, n, port):
    """torchrun command that re-executes this script with one rank per GPU."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
            "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *argv]


def relaunch(args, argv):
    """--gpus N > 1 outside torchrun: check the devices, then run N ranks."""
    if args.impl == "ours":
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} but only {have} CUDA device(s) visible", file=sys.stderr)
            return 2
    cmd = launch_command(argv, args.gpus, _free_port())
    print("bench.py: " + " ".join(cmd), file=sys.stderr, flush=True)
    return subprocess.run(cmd).returncode


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    args = parse(argv)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args, argv)
    rank = _env_int("RANK", 0)
    world = _env_int("WORLD_SIZE", 1)
    local = _env_int("LOCAL_RANK", 0)
    if args.config is None:
        args.config = "cfg2" if world == 1 else "cfg3"
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    dist = None
    force_comm = os.environ.get("CDR_FORCE_COMM") == "1" and "RANK" in os.environ  # test hook
    if world > 1 or force_comm:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2103_15208_b200 import api

    seed = 1
    scene, gids, cfg, total_views = build_workload(args.config, rank, world, args.views)
    spp = cfg["spp"]
    r = api.Renderer(local, scene, view_ids=gids)
    if world > 1 or os.environ.get("CDR_FORCE_COMM") == "1":
        # one NCCL communicator per GPU for the gradient all-reduce inside
        # cdr_loss_grad; the 128-byte id travels over torch.distributed
        uid = [api.Renderer.nccl_unique_id() if rank == 0 else None]
        if dist is not None:
            dist.broadcast_object_list(uid, src=0)
        r.comm_init(uid[0], world, rank)
        nranks, crank = r.comm_info()
        print(f"[bench] rank {rank}: NCCL communicator of {nranks} ranks, this rank {crank} on cuda:{local}",
              file=sys.stderr, flush=True)
        if nranks != world:
            raise RuntimeError(f"NCCL communicator has {nranks} ranks, expected {world}")
    # targets: the perturbed scene rendered by the same engine (gradcheck.cpp:49-73)
    from paper_2103_15208_b200 import scenes as S
    tr = api.Renderer(local, S.perturbed_target_scene(scene), view_ids=gids)
    for k in range(len(scene.cameras)):
        img, _, _ = tr.render(k, api.RenderSettings(spp=spp, seed=seed + 0x7A9), want_hits=False)
        r.set_target(k, img)
    tr.close()
    lay = api.param_layout(scene)
    st = api.RenderSettings(spp=spp, seed=seed)
    views = np.arange(len(scene.cameras), dtype=np.int32)

    stream = torch.cuda.ExternalStream(r.stream(), device=torch.device("cuda", local))
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{local}")

    def barrier():
        torch.cuda.synchronize(local)
        if dist is not None:
            dist.barrier()

    for _ in range(args.warmup):
        r.loss_grad(views, st, lay, device_only=True)
    barrier()
    clocks = clock_sampler(local) if rank == 0 else None
    evs = []
    stats = []
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            flush.zero_()  # L2 flush (256 MB > 126 MB L2), outside the timed window
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
        _, _, s, _ = r.loss_grad(views, st, lay, device_only=True)
        with torch.cuda.stream(stream):
            b.record(stream)
        evs.append((a, b))
        stats.append(s.as_dict())
    barrier()
    clk = clocks.stop() if clocks else None
    ms_steps = [a.elapsed_time(b) for a, b in evs]
    t_local = sum(ms_steps)
    t = torch.tensor([t_local], dtype=torch.float64, device=f"cuda:{local}")
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_max = float(t.item())
    samples_rank = sum(c.width * c.height for c in scene.cameras) * spp
    samples_all = sum(cfg["image"] ** 2 for _ in range(total_views)) * spp
    total_samples = samples_all * args.steps
    value = total_samples / (t_max / 1e3) / 1e6

    # ---- roofline of the dominant kernel (fused trace/shade/loss/interior)
    s0 = stats[-1]
    ms_shade = statistics.mean(x["ms_render"] - x["ms_trace"] for x in stats)
    n_px, n_samp = s0["pixels"], s0["shaded_samples"]  # empty beam tiles touch no hit cache
    n_hit, n_adj = s0["hit_samples"], s0["adjoint_samples"]
    # SURVEY §8(d) per-unit algorithmic bytes (fp32 texels and texel-gradient RMW)
    algo_bytes = 80 * n_px + 4 * n_samp + 316 * n_hit + 512 * n_adj
    # the same traffic at this implementation's storage (32-B texel records,
    # fp64 texel-gradient accumulator): reported beside it, not as `achieved`
    stored_bytes = 80 * n_px + 4 * n_samp + 332 * n_hit + 736 * n_adj
    pk, pk_kind = peaks()
    achieved = algo_bytes / (ms_shade / 1e3) / 1e9
    roof = {"kernel": "k_render<shade,loss,interior> (fused shading + loss + interior scatter)",
            "bound": "hbm", "achieved": achieved,
            "peak": pk["hbm_gbs"], "peak_source": pk_kind, "unit": "GB/s", "frac": achieved / pk["hbm_gbs"],
            "traffic": None, "algorithmic_bytes_per_launch": algo_bytes,
            "byte_model": "SURVEY §8(d): 80*N_px + 4*N_shaded + 316*N_hit + 512*N_adj (DESIGN.md §4)",
            "storage_bytes_per_launch": stored_bytes,
            "storage_frac": stored_bytes / (ms_shade / 1e3) / 1e9 / pk["hbm_gbs"],
            "ms_per_launch": ms_shade, "share_of_step": ms_shade / statistics.mean(ms_steps)}
    # DRAM traffic of the same kernel at THIS config, from the committed ncu
    # capture of this step (profiles/profile_step.py --bench-step,
    # profiles/r2/per_kernel_<cfg>_step.json);
    # configs without a capture report null rather than a scaled figure
    traffic_file = os.path.join(ROOT, "profiles", "r2", f"per_kernel_{args.config}_step.json")
    roof["traffic"] = None
    roof["traffic_source"] = f"no ncu capture of {args.config}"
    if os.path.exists(traffic_file) and args.views is None and world == 1:
        try:
            kern = json.load(open(traffic_file))["kernels"]
            # the step's fused instance (fp32 texel records: synthetic maps)
            kr = max((v for k, v in kern.items() if k.startswith("k_render<1, 1, 1,") and k.endswith(", 0>")),
                     key=lambda v: v["ms"])
            roof["traffic"] = 1e6 * (kr["dram_read_MB"] + kr["dram_write_MB"])
            roof["traffic_source"] = (f"ncu dram__bytes_read.sum + dram__bytes_write.sum of the fused k_render "
                                      f"in this step at {args.config}, {os.path.relpath(traffic_file, ROOT)}")
            # what HBM actually moved per launch, over this run's kernel time: the
            # algorithmic fraction above is served mostly from L2 (mesh, BVH, maps)
            roof["dram_GBps"] = roof["traffic"] / (ms_shade / 1e3) / 1e9
            roof["dram_frac"] = roof["dram_GBps"] / pk["hbm_gbs"]
        except Exception as e:  # noqa: BLE001
            roof["traffic_source"] = f"unreadable capture: {e}"

    # the boundary stage against the same roofline: SURVEY §8(d)'s 970 B per
    # active boundary sample (segment record, CDF search, adjoint, two probe
    # shadings, vertex RMW) over the stage's event-timed window. The window
    # holds the probes and deposits (k_boundary); the sampling kernels
    # (k_bsample / k_bscan / k_bscatter) run on the side stream beside the
    # render, so `frac` is an upper bound and `frac_serial` adds their
    # serialised ncu time from this config's step capture when there is one.
    ms_bnd_stage = statistics.mean(x["ms_boundary"] for x in stats)
    bnd_bytes = 970 * s0["boundary_active"]
    bnd = {"kernel": "k_boundary (probes + deposits)", "bound": "hbm", "unit": "GB/s",
           "bytes_per_active_sample": 970, "active_samples": s0["boundary_active"],
           "algorithmic_bytes": bnd_bytes, "ms": ms_bnd_stage,
           "achieved": bnd_bytes / (ms_bnd_stage / 1e3) / 1e9 if ms_bnd_stage > 0 else None,
           "peak": pk["hbm_gbs"]}
    bnd["frac"] = bnd["achieved"] / pk["hbm_gbs"] if bnd["achieved"] else None
    try:
        kern = json.load(open(traffic_file))["kernels"] if os.path.exists(traffic_file) else {}
        ms_samp = sum(kern[k]["ms"] for k in ("k_bsample", "k_bscan", "k_bscatter") if k in kern)
        if ms_samp > 0 and args.views is None and world == 1:
            bnd["ms_sampling_serial"] = ms_samp
            bnd["frac_serial"] = bnd_bytes / ((ms_bnd_stage + ms_samp) / 1e3) / 1e9 / pk["hbm_gbs"]
    except Exception:  # noqa: BLE001
        pass

    # traversal throughput (latency-bound, reported as Mrays/s):
    # primary rays = samples of non-empty beam tiles (k_tile_lists + k_trace),
    # boundary probe rays = 2 per active edge sample (k_bsample..k_boundary)
    ms_trace = statistics.mean(x["ms_trace"] for x in stats)
    ms_bnd = statistics.mean(x["ms_boundary"] for x in stats)
    traversal = {"primary_Mrays_per_s": s0["shaded_samples"] / (ms_trace / 1e3) / 1e6,
                 "primary_rays": s0["shaded_samples"], "ms_visibility": ms_trace,
                 "probe_Mrays_per_s": 2 * s0["boundary_active"] / (ms_bnd / 1e3) / 1e6,
                 "probe_rays": 2 * s0["boundary_active"], "ms_boundary": ms_bnd,
                 "note": "per rank; visibility = candidate lists + trace; boundary = probes + deposits (the sampling kernels run on the side stream beside the render)"}

    # ---- e2e: host buffers through the C-ABI
    e2e = None
    if not args.no_e2e:
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
        pos_h = pin(scene.mesh.positions)
        d_h, s_h, r_h = pin(scene.diffuse), pin(scene.specular), pin(scene.roughness)
        g_h = pin(np.zeros(lay["total"]))
        npx = sum(c.width * c.height for c in scene.cameras)
        rgb_h, msk_h = pin(np.zeros(3 * npx)), pin(np.zeros(npx))

        def timed_e2e(staged, images):
            # one step = positions + 3 maps up, the loss call, the gradient
            # (+ the K rendered images and masks) and the loss terms down
            barrier()
            t0 = time.perf_counter()
            for _ in range(args.steps):
                if staged:  # cdr_stage_params: read by the loss call, copies overlapped with its kernels
                    r.stage_params(pos_h, (d_h, s_h, r_h))
                else:       # separate synchronous uploads before the call
                    r.update_positions(pos_h)
                    r.set_textures(d_h, s_h, r_h)
                r.loss_grad(views, st, lay, grad=g_h, overwrite=True,  # fresh gradient, as total_loss
                            rendered_out=rgb_h if images else None, mask_out=msk_h if images else None)
            barrier()
            te = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=f"cuda:{local}")
            if dist is not None:
                dist.all_reduce(te, op=dist.ReduceOp.MAX)
            return float(te.item())

        h2d = pos_h.nbytes + d_h.nbytes + s_h.nbytes + r_h.nbytes
        d2h = g_h.nbytes + 16
        dt = timed_e2e(True, False)
        e2e = {"value": total_samples / dt / 1e6, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": 1e3 * dt / args.steps,
               "what": "cdr_stage_params + cdr_loss_grad with pinned host buffers: positions + 3 maps up, "
                       "gradient + loss down (maps up beside the visibility pass, map gradient down beside "
                       "the boundary pass)"}
        dt = timed_e2e(False, False)
        e2e["separate_uploads"] = {"value": total_samples / dt / 1e6, "ms_per_step": 1e3 * dt / args.steps,
                                   "what": "cdr_update_positions + cdr_set_textures, then cdr_loss_grad"}
        # the same with total_loss's rendered images and masks (the K Images of
        # TotalLossResult, losses.cpp:259) downloaded into pinned buffers too
        dt = timed_e2e(True, True)
        e2e["with_rendered_images"] = {
            "value": total_samples / dt / 1e6, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h + rgb_h.nbytes + msk_h.nbytes), "ms_per_step": 1e3 * dt / args.steps}

    # ---- the four mesh/material regularisers of total_loss (losses.cpp:272-292)
    # at the reference's default weights: texture-size work, not per sample, so
    # timed on their own (device events on the library stream)
    regs = None
    if rank == 0:
        lw = api.LossWeights()
        r.regularisers(lw, lay, device_only=True)
        rev = []
        for _ in range(max(3, args.steps)):
            with torch.cuda.stream(stream):
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(stream)
            vals, _ = r.regularisers(lw, lay, device_only=True)
            with torch.cuda.stream(stream):
                b.record(stream)
            rev.append((a, b))
        torch.cuda.synchronize(local)
        regs = {"ms": statistics.median(a.elapsed_time(b) for a, b in rev), "values": vals,
                "texels": int(scene.diffuse.shape[0] * scene.diffuse.shape[1]), "tris": scene.mesh.T,
                "weights": "LossWeights defaults (losses.hpp:14-23)"}
        if world == 1 and not args.no_cpu_baseline:
            try:
                from oracle.pyoracle import RefLib
                ref = RefLib(scene)
                t0 = time.perf_counter()
                ref.regularisers((lw.normal, lw.edge, lw.spec, lw.roug, lw.sigma1, lw.sigma2))
                regs["cpu_ms"] = 1e3 * (time.perf_counter() - t0)
                regs["cpu_kind"] = "reference (oracle/_ref), 1 thread: the reference functions are serial"
            except Exception as e:  # noqa: BLE001 — the CPU leg is optional
                regs["cpu_ms"] = None
                regs["cpu_kind"] = f"unavailable: {e}"

    # ---- ms per optimisation iteration (the metric's second half), resident:
    # total_loss with all six terms (LossWeights defaults) -> adam_step ->
    # robust_evolve, every step on the device, only scalars back to the host
    iteration = None
    if not args.no_iteration:
        diag = float(np.linalg.norm(np.ptp(scene.mesh.positions, axis=0)))
        acfg = api.AdamConfig(lr_positions=1e-3 * diag)  # the plan's scaling (optimize.hpp:15)
        r.adam_init(acfg, lay)
        lw = api.LossWeights()

        def one_iteration(parts):
            t0 = time.perf_counter()
            bd, _ = r.total_loss_device(views, st, lay, lw)
            t1 = time.perf_counter()
            r.adam_step(want_displacement=False)
            t2 = time.perf_counter()
            sc, _ = r.evolve(want_positions=False)
            t3 = time.perf_counter()
            parts.append((t1 - t0, t2 - t1, t3 - t2, sc, bd["total"]))

        warm = []
        for _ in range(2):
            one_iteration(warm)
        barrier()
        parts = []
        for _ in range(max(3, args.steps)):
            one_iteration(parts)
        barrier()
        med = lambda i: 1e3 * statistics.median(p[i] for p in parts)
        tot = [1e3 * (p[0] + p[1] + p[2]) for p in parts]
        ti = torch.tensor([statistics.median(tot)], dtype=torch.float64, device=f"cuda:{local}")
        if dist is not None:
            dist.all_reduce(ti, op=dist.ReduceOp.MAX)
        iteration = {"ms": float(ti.item()), "parts_ms": {"total_loss": med(0), "adam_step": med(1), "evolve": med(2)},
                     "evolve_scales": [p[3] for p in parts], "loss_total": [p[4] for p in parts],
                     "iterations": len(parts), "timing": "host wall clock around each synchronous call",
                     "what": "total_loss (rendering + Laplacian + 4 regularisers, LossWeights defaults) -> "
                             "adam_step + apply -> robust_evolve, resident on the device"}
        iteration["ms_each"] = [round(x, 3) for x in tot]
    cpu = None
    cb = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = cpu_baseline_sample(scene, spp, seed, lay, os.cpu_count() or 1, label=args.config)
        cpu = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
    if iteration is not None:
        if cb is not None:  # the reference's iteration, extrapolated from the bounded sample
            per_view_s = cb["seconds"] * (cfg["image"] ** 2 * spp) / cb["samples"]
            ref_ms = per_view_s * total_views * 1e3 + ((regs or {}).get("cpu_ms") or 0.0)
            iteration["reference_ms_extrapolated"] = ref_ms
            iteration["reference_basis"] = (f"mean total_loss time per view of the {CPU_SUBSET}-view subset x "
                                            f"{total_views} views ({cb['cores']} threads) + the serial regularisers; "
                                            "adam/evolve not included")

    if rank == 0:
        stages = {k: statistics.mean(x[k] for x in stats) for k in
                  ("ms_prepare", "ms_trace", "ms_render", "ms_silhouette", "ms_boundary", "ms_finalize", "ms_total")}
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True,
                "scaling": cfg["scaling"], "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": workload_text(args.config, cfg, total_views), "name": args.config,
                           "views_per_gpu": len(scene.cameras), "spp": spp,
                           "samples_per_step": samples_all, "parallelism": f"views sharded x{world}",
                           "l2": "flushed (256 MB write) before every timed step; step working set ~2 GB"},
                "roofline": roof, "boundary_roofline": bnd, "cpu_baseline": cpu, "e2e": e2e, "regularisers": regs, "iteration": iteration,
                "traversal": traversal,
                "gpu_launches": int(sum(x["kernel_launches"] for x in stats)),
                "clocks": clk, "stages_ms": stages,
                "counters": {k: s0[k] for k in ("pixels", "samples", "hit_samples", "adjoint_samples",
                                                "boundary_samples", "boundary_active", "segments",
                                                "beam_fallback_tiles", "shaded_samples")}}
        print(json.dumps(line), flush=True)
    r.close()
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
