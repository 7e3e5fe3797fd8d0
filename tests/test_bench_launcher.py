"""bench.py's multi-GPU launcher and the view-shard arithmetic (CPU).

`python bench.py --gpus N` outside torchrun re-executes itself under
torch.distributed.run with N ranks (one per GPU) and refuses to run with fewer
than N devices; the default workload at N > 1 is cfg3 split over the ranks
(strong scaling). The reference arm runs the same launcher (rank 0 prints)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2103_15208_b200.shard import shard_views, weak_views  # noqa: E402


def test_launch_command_is_torchrun_one_rank_per_gpu():
    cmd = bench.launch_command(["--gpus", "4", "--steps", "3"], 4, 29555)
    assert cmd[:3] == [sys.executable, "-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--nnodes=1" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[cmd.index("--master-port") + 1] == "29555"
    assert cmd[-3:] == ["--gpus", "4", "--steps", "3"][-3:]
    assert os.path.basename(cmd[cmd.index("--master-port") + 2]) == "bench.py"


def test_too_few_devices_exits_nonzero():
    import torch
    n = torch.cuda.device_count()
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(max(2, n + 1))],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode != 0
    assert "CUDA device" in r.stderr


@pytest.mark.parametrize("n_views,world", [(100, 1), (100, 2), (100, 4), (100, 8), (400, 8), (50, 3), (4, 8)])
def test_strong_shards_cover_every_view_once(n_views, world):
    got = [g for r in range(world) for g in shard_views(n_views, world, r)]
    assert got == list(range(n_views))
    sizes = [len(shard_views(n_views, world, r)) for r in range(world)]
    assert max(sizes) == -(-n_views // world)


def test_weak_shards_are_disjoint_blocks():
    blocks = [weak_views(50, r) for r in range(8)]
    flat = [g for b in blocks for g in b]
    assert flat == list(range(400))


def test_default_config_per_world():
    # cfg2 (configs[1], weak) at one GPU, cfg3 (configs[2], strong) at N > 1
    assert bench.CONFIGS["cfg2"]["scaling"] == "weak" and bench.CONFIGS["cfg3"]["scaling"] == "strong"
    assert bench.CONFIGS["cfg3"]["views"] == 100 and bench.CONFIGS["cfg3"]["tex"] == 1024


@pytest.mark.ref
def test_reference_arm_through_the_launcher():
    """--gpus 2 relaunches under torchrun over gloo-free CPU ranks: rank 0
    alone runs the reference and prints one line with n_gpus 2."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "1", "--warmup", "0", "--config", "cfg1"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["config"]["name"] == "cfg1"
    assert d["cpu_baseline"]["kind"] == "reference"
