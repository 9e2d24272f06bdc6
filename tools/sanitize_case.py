"""Small end-to-end evaluation for compute-sanitizer (memcheck / racecheck / synccheck):
cfg2 (N = 1e4, P = 100) through the public API and the device-resident step, a
forced neighbour-row overflow (overflow kernel), the z-split phases and the
fused tile short range -- every kernel family of the evaluation once."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2403_01521_b200 as pk  # noqa: E402
from paper_2403_01521_b200.configs import make_workload  # noqa: E402
from paper_2403_01521_b200.engine import DeviceEvaluator, get_engine  # noqa: E402

wl = make_workload(sys.argv[1] if len(sys.argv) > 1 else "cfg2")
soe = pk.build_soe_contour(wl.m)
params = wl.params()
sampler = pk.ModeSampler(wl.alpha, wl.box, seed=wl.seed)
bd, f = pk.rb_energy_forces(wl.system, wl.box, params, soe, sampler, wl.P)
print("rb_energy_forces total", bd.total)
ev = DeviceEvaluator(wl.system, wl.box, params, soe, P=wl.P, seed=wl.seed)
ev.warmup()
ev.step()
pos2 = torch.as_tensor(wl.system.pos).clone()
pos2[:, 2] = 0.4 * wl.box.lz + 0.2 * pos2[:, 2]       # squeeze: rows overflow
ev.set_positions(pos2.to(ev.eng.device))
ev.step()
torch.cuda.synchronize()
print("squeezed status", ev.status())
# z-split phases of two emulated ranks on one context each
eng = get_engine()
from paper_2403_01521_b200 import _native  # noqa: E402
from paper_2403_01521_b200.engine import Engine  # noqa: E402
dev = eng.device
pos = torch.as_tensor(wl.system.pos).to(dev)
q = torch.as_tensor(wl.system.charge).to(dev)
modes = torch.as_tensor(sampler.batch(wl.P)).to(dev)
cnt = int(_native.load().slab_zsplit_exchange_doubles(wl.P, wl.m, 1))
engines = [Engine(dev) for _ in range(2)]
x = [torch.zeros(cnt, dtype=torch.float64, device=dev) for _ in range(2)]
args = (pos, q, wl.box, wl.alpha, params.r_c, soe, modes, 0.37, 1.5)
for r in range(2):
    engines[r].evaluate(*args, shard=(r, 2), shard_mode=1, phase=1, xchg=x[r])
xa = torch.cat(x)
for r in range(2):
    engines[r].evaluate(*args, shard=(r, 2), shard_mode=1, phase=2, xchg=xa)
torch.cuda.synchronize()
os.environ["SLAB_SHORT_TILE"] = "1"
big = make_workload("cfg5_1e5")
u, _ = pk.short_range_energy_forces(big.system, big.box, big.alpha, big.params().r_c)
print("tile short range", u)
print("SANITIZE_CASE_DONE")
