"""MD throughput of the device-resident engine (md.run_simulation path).

    python tools/md_bench.py [N] [steps] [solver]

Jittered-lattice +-1 system at density 0.1 in a slab box (Lx = Ly = 2 Lz),
Langevin thermostat, rbse2d (P = batch_size) or soewald2d, WCA core + walls.
Reports steps/s and the per-step device time split (torch.profiler)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2403_01521_b200 as pk  # noqa: E402
from paper_2403_01521_b200 import md  # noqa: E402


def lattice_system(n, seed=0):
    lz = (n / (4 * 0.1)) ** (1 / 3)
    box = pk.BoxGeometry(2 * lz, 2 * lz, lz)
    m = int(np.ceil((n / 4) ** (1 / 3)))
    g = np.stack(np.meshgrid((np.arange(2 * m) + 0.5) / (2 * m), (np.arange(2 * m) + 0.5) / (2 * m),
                             (np.arange(m) + 0.5) / m, indexing="ij"), -1).reshape(-1, 3)
    rng = np.random.default_rng(seed)
    g = g[rng.permutation(len(g))[:n]] * [box.lx, box.ly, box.lz]
    g += rng.uniform(-0.2, 0.2, g.shape)
    q = np.where(np.arange(n) % 2 == 0, 1.0, -1.0)
    return pk.make_system(q, np.ones(n), g, box=box), box


def main():
    n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
    solver = sys.argv[3] if len(sys.argv) > 3 else "rbse2d"
    s, box = lattice_system(n)
    opts = md.MDOptions(dt=0.002, n_steps=steps, thermostat="langevin", solver=solver,
                        alpha=(n / box.volume) ** (1 / 3) if hasattr(box, "volume") else
                        (n / (box.lx * box.ly * box.lz)) ** (1 / 3),
                        s=4.0, soe_size=16, batch_size=100, sample_every=steps, seed=1)
    md.run_simulation(s, box, md.MDOptions(**{**opts.__dict__, "n_steps": 2,
                                                 "sample_every": 2}))
    torch.cuda.synchronize()
    t = time.perf_counter()
    res = md.run_simulation(s, box, opts)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"N={n} {solver}: {steps} steps in {dt:.3f} s -> {steps / dt:.1f} steps/s "
          f"({1e3 * dt / steps:.2f} ms/step incl. setup and 2 samples); "
          f"K/N = {res.kinetic[-1] / n:.3f}")
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        md.run_simulation(s, box, md.MDOptions(**{**opts.__dict__, "n_steps": 5,
                                                     "sample_every": 5}))
        torch.cuda.synchronize()
    rows = sorted(((e.device_time_total / 1e3 / 5, e.key) for e in prof.key_averages()
                   if e.device_time_total > 0), reverse=True)[:12]
    for ms, k in rows:
        print(f"  {ms:8.3f} ms/step  {k[:90]}")


if __name__ == "__main__":
    main()
