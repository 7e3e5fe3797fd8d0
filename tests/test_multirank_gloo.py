"""View-sharded data parallelism, host logic on CPU: world_size 2 over gloo.

Each rank evaluates its shard of views (global view ids as RNG keys) with the
CPU oracle; the gradient and loss terms are all-reduced; the result must equal
the single-process evaluation of all views. The GPU path runs the same
sharding with the library's NCCL all-reduce (bench.py under torchrun)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2103_15208_b200 import scenes as S
from paper_2103_15208_b200.shard import laplacian_weight, shard_views


def _scene():
    return S.make_scene(S.blob(6), 16, 5, 24)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.pyoracle import Oracle, layout_for, settings
    from tests.scenes_util import targets_for
    full = _scene()
    tg_all = targets_for(full, 4, 2, Oracle)
    gids = shard_views(len(full.cameras), world, rank)
    shard = S.Scene(full.mesh, full.diffuse, full.specular, full.roughness, [full.cameras[g] for g in gids])
    o = Oracle(shard, view_ids=gids)
    lay = layout_for(full)
    loss, g, _ = o.loss_grad(tg_all[gids], settings(4, 2), lay, lam_lap=0.1 * laplacian_weight(rank))
    t = torch.from_numpy(np.concatenate([loss, g]))
    dist.all_reduce(t)
    if rank == 0:
        np.save(out_path, t.numpy())
    dist.destroy_process_group()


def test_two_rank_view_sharding_equals_single_process(tmp_path):
    out = str(tmp_path / "r.npy")
    mp.start_processes(_worker, args=(2, _free_port(), out), nprocs=2, join=True, start_method="spawn")
    red = np.load(out)
    from oracle.pyoracle import Oracle, layout_for, settings
    from tests.scenes_util import targets_for
    full = _scene()
    tg = targets_for(full, 4, 2, Oracle)
    loss, g, _ = Oracle(full).loss_grad(tg, settings(4, 2), layout_for(full), lam_lap=0.1)
    np.testing.assert_allclose(red[:2], loss, rtol=1e-12)
    np.testing.assert_allclose(red[2:], g, rtol=1e-9, atol=1e-12 * np.abs(g).max())
