"""Multi-GPU code path of ``DeviceEvaluator`` with world size 2.

Two processes drive the REAL sharded step -- their share of the modes (or of the
z-sorted chunk range) and of the short-range homes, the exchange and the one
all-reduce -- on the one GPU this suite has, over a gloo group (host-staged
collectives: no kernel of one rank waits on a kernel of the other).  The summed
result must match the reference's own outputs (tests/golden) at the north-star
tolerances.  Rendezvous on 127.0.0.1.
"""

import os
import socket

import numpy as np
import pytest

from helpers import load_golden

pytestmark = pytest.mark.gpu

E_TOL = 1e-10
F_TOL = 1e-9


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, name, mode, out, graph=False):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_2403_01521_b200 as pk
    from paper_2403_01521_b200.configs import make_workload
    from paper_2403_01521_b200.engine import DeviceEvaluator
    g = load_golden(name)
    wl = make_workload(name)
    soe = pk.build_soe_contour(wl.m)
    ev = DeviceEvaluator(wl.system, wl.box, wl.params(), soe, P=int(g["P"]), H=float(g["H"]),
                         c_q=float(g["c_q"]), modes=g["modes"], sample=False, rank=rank,
                         world=world, group=dist.group.WORLD, shard_mode=mode)
    ev.warmup()
    if graph:  # the rank's local parts as CUDA graphs, collectives between replays
        ev.capture()
    e, f = ev.step()
    torch.cuda.synchronize()
    if rank == 0:
        np.savez(out, energy=e.cpu().numpy(), forces=f.cpu().numpy(), status=ev.status())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("graph", [False, True])
@pytest.mark.parametrize("mode", ["modes", "zsplit"])
@pytest.mark.parametrize("name", ["small_2000", "cfg4"])
def test_two_rank_device_evaluator_matches_reference(tmp_path, name, mode, graph):
    import torch.multiprocessing as mp
    g = load_golden(name)
    out = str(tmp_path / "rank0.npz")
    mp.start_processes(_worker, args=(2, _free_port(), name, mode, out, graph), nprocs=2,
                       join=True, start_method="spawn")
    r = np.load(out)
    e, f = r["energy"], r["forces"]
    assert int(r["status"]) == 0
    for val, key in zip(e[:5], ("u_s", "u_l_k", "u_l_0", "u_self", "u_ps")):
        ref = float(g[key])
        assert abs(val - ref) <= E_TOL * max(abs(ref), 1e-300), (key, val, ref)
    tot = e[0] + e[1] + e[2] - e[3] + e[4]
    assert abs(tot - float(g["total"])) <= E_TOL * abs(float(g["total"]))
    fs = f[g["sample_idx"]] if "sample_idx" in g else f
    assert np.max(np.abs(fs - g["forces"])) <= F_TOL * float(g["fmax"])
