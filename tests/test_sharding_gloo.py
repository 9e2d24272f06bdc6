"""CPU, world_size 2 over gloo: the multi-GPU decomposition of one evaluation.

Each rank computes exactly the share the device path assigns to it
(paper_2403_01521_b200.sharding: its mode slice, its short-range home
particles of the stable cell order, lead-rank-only k = 0 mode and constants),
here with the C oracle; ONE all_reduce of the packed (3N + 5) buffer must give
the unsharded evaluation.  Rendezvous on 127.0.0.1.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _shard_eval(rank, world, name):
    from oracle import oracle as O
    from paper_2403_01521_b200.configs import make_workload
    from paper_2403_01521_b200.sharding import home_range, is_lead, mode_slice
    from helpers import load_golden
    g = load_golden(name)
    wl = make_workload(name)
    n, P = wl.n, int(g["P"])
    soe_w, soe_s = g["soe_w"], g["soe_s"]
    rc = wl.params().r_c
    t0, t1 = mode_slice(P, rank, world)
    h0, h1 = home_range(n, rank, world)
    perm = O.sort_perm(wl.system.pos[:, 2], wl.box.lz)
    xs, ys, zs = (wl.system.pos[perm, i] for i in range(3))
    qs = wl.system.charge[perm]
    cv = O.rb_commonv(float(g["H"]), P, wl.alpha)
    u_k, fs = O.fourier_sweep(xs, ys, zs, qs, g["modes"][t0:t1], cv[t0:t1], soe_w, soe_s,
                             wl.alpha, wl.box.area)
    f = np.zeros((n, 3))
    f[perm] = fs
    u_s, f_s, _ = O.short_range_home(wl.system.pos, wl.system.charge, wl.box, wl.alpha, rc, h0,
                                     h1)
    f += f_s
    e = np.zeros(5)
    e[0], e[1] = u_s, u_k
    if is_lead(rank):
        # k = 0 mode + constants: the full evaluation minus its nonzero-mode and
        # short-range parts (oracle_energy_forces with no modes, short range zero)
        e_all, f_all, _ = O.energy_forces(wl.system.pos, wl.system.charge, wl.box, wl.alpha, rc,
                                          np.zeros((0, 3)), np.zeros(0), float(g["c_q"]), soe_w,
                                          soe_s)
        _, f_s_all, _ = O.short_range(wl.system.pos, wl.system.charge, wl.box, wl.alpha, rc)
        e[1] += e_all[1]
        e[2:] = e_all[2:]
        f += f_all - f_s_all
    return np.concatenate([f.ravel(), e])


def _worker(rank, world, port, name, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    buf = torch.from_numpy(_shard_eval(rank, world, name))
    dist.all_reduce(buf, op=dist.ReduceOp.SUM)   # the single collective of the step
    if rank == 0:
        np.save(out, buf.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["small_600", "small_2000"])
def test_two_rank_decomposition_equals_single_rank(tmp_path, name):
    from helpers import load_golden
    out = str(tmp_path / "red.npy")
    mp.start_processes(_worker, args=(2, _free_port(), name, out), nprocs=2, join=True,
                       start_method="spawn")
    red = np.load(out)
    g = load_golden(name)
    n = len(g["forces"])
    f, e = red[:3 * n].reshape(n, 3), red[3 * n:]
    for val, key in zip(e, ("u_s", "u_l_k", "u_l_0", "u_self", "u_ps")):
        ref = float(g[key])
        assert abs(val - ref) <= 1e-12 * max(abs(ref), 1.0), (key, val, ref)
    assert np.max(np.abs(f - g["forces"])) <= 1e-12 * float(g["fmax"])


def test_slices_partition_the_work():
    from paper_2403_01521_b200.sharding import home_range, mode_slice
    for P, n, w in [(100, 999_999, 8), (7, 10, 3), (200, 100_000, 4)]:
        ms = [mode_slice(P, r, w) for r in range(w)]
        hs = [home_range(n, r, w) for r in range(w)]
        assert ms[0][0] == 0 and ms[-1][1] == P and hs[0][0] == 0 and hs[-1][1] == n
        assert all(ms[r][1] == ms[r + 1][0] for r in range(w - 1))
        assert all(hs[r][1] == hs[r + 1][0] for r in range(w - 1))
