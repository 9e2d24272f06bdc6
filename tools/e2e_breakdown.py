"""Host-side breakdown of one rb_energy_forces call (public API, pinned inputs)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2403_01521_b200 as pk  # noqa: E402
from paper_2403_01521_b200 import rbse2d, soewald2d  # noqa: E402
from paper_2403_01521_b200.configs import make_workload  # noqa: E402
from paper_2403_01521_b200.engine import pinned_like  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
wl = make_workload(name)
soe = pk.build_soe_contour(wl.m)
params = wl.params()
H = rbse2d.normalization_H(wl.alpha, wl.box)
c_q = rbse2d.charge_term_sum(wl.alpha, wl.box, float(np.sum(wl.system.charge ** 2)))
s = pk.make_system(wl.system.charge, wl.system.mass, wl.system.pos, box=wl.box)
s.pos = pinned_like(wl.system.pos)
s.charge = pinned_like(wl.system.charge)
smp = rbse2d.ModeSampler(wl.alpha, wl.box, seed=wl.seed)

if "--with-evaluator" in sys.argv:
    from paper_2403_01521_b200.engine import DeviceEvaluator
    ev = DeviceEvaluator(wl.system, wl.box, params, soe, P=wl.P, H=H, c_q=c_q, seed=wl.seed)
    ev.warmup()
    for _ in range(5):
        ev.step()
    torch.cuda.synchronize()
T = {}
orig = {}


def wrap(mod, fn):
    f = getattr(mod, fn)
    orig[(mod, fn)] = f

    def g(*a, **k):
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = f(*a, **k)
        torch.cuda.synchronize()
        T[fn] = T.get(fn, 0.0) + time.perf_counter() - t
        return r
    setattr(mod, fn, g)


for _ in range(3):
    pk.rb_energy_forces(s, wl.box, params, soe, smp, wl.P, H=H, c_q=c_q)
torch.cuda.synchronize()
K = 10
t = time.perf_counter()
for _ in range(K):
    pk.rb_energy_forces(s, wl.box, params, soe, smp, wl.P, H=H, c_q=c_q)
torch.cuda.synchronize()
print(f"rb_energy_forces: {1e3 * (time.perf_counter() - t) / K:.3f} ms/call (no instrumentation)")
wrap(smp.__class__, "batch")
wrap(rbse2d, "device_evaluate")
from paper_2403_01521_b200 import engine  # noqa: E402
wrap(engine, "to_device")
wrap(engine, "host_result")
wrap(engine.Engine, "evaluate")
for _ in range(K):
    pk.rb_energy_forces(s, wl.box, params, soe, smp, wl.P, H=H, c_q=c_q)
for k, v in T.items():
    print(f"  {k:18s} {1e3 * v / K:8.3f} ms/call (synchronised)")
