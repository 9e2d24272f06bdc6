"""bench.py's multi-GPU launcher (CPU): ``--gpus N`` outside torchrun starts N
ranks of itself under torch.distributed.run (one process per GPU on a B200 box)."""

import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_gpus_2_spawns_two_ranks():
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "2",
                          "--probe"], capture_output=True, text=True, env=env, timeout=300,
                         check=True).stdout
    lines = [json.loads(l) for l in out.splitlines() if l.startswith("{")]
    assert sorted(d["rank"] for d in lines) == [0, 1]
    assert all(d["world"] == 2 for d in lines)


def test_launch_command_is_torchrun_with_nproc():
    sys.path.insert(0, REPO)
    import bench
    cmd = bench.launch_command(["--gpus", "8", "--steps", "5"], 8, 12345)
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=8" in cmd and "--master-addr=127.0.0.1" in cmd
    assert cmd[-4:] == ["--gpus", "8", "--steps", "5"]


import pytest  # noqa: E402


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["modes", "zsplit"])
def test_multi_rank_bench_path_prints_the_contract_line(mode):
    """The whole ``--gpus 2`` bench path -- launcher, per-rank CUDA graphs with the
    collectives between replays, the scan timing, the sharded e2e -- on a one-GPU
    box: both ranks on cuda:0 over gloo (SLAB_BENCH_BACKEND, test only; the
    timings are not scaling numbers).  Rank 0 prints one contract JSON line."""
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    env["SLAB_BENCH_BACKEND"] = "gloo"
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "2",
                          "--steps", "1", "--warmup", "3", "--shard-mode", mode,
                          "--no-cpu-baseline"], capture_output=True, text=True, env=env,
                         timeout=900, check=True).stdout
    lines = [json.loads(l) for l in out.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = lines[0]
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["status"] == 0
    assert d["config"]["cuda_graph"] is True
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    assert 0 < d["roofline"]["frac"] < 1
