"""Debug: full evaluation at a golden config -- host entry (forked short range)
against the device entry, energies vs the reference."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2403_01521_b200 as pk
from paper_2403_01521_b200.configs import make_workload
from paper_2403_01521_b200.engine import get_engine
from paper_2403_01521_b200.rbse2d import _rb_commonv
from helpers import StubSampler

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5_1e7"
g = dict(np.load(f"tests/golden/{name}.npz"))
wl = make_workload(name)
soe = pk.build_soe_contour(wl.m)
params = wl.params()
P = int(g["P"])
bd, f = pk.rb_energy_forces(wl.system, wl.box, params, soe, StubSampler(g["modes"]), P,
                            H=float(g["H"]), c_q=float(g["c_q"]))
keys = ("u_s", "u_l_k", "u_l_0", "u_self", "u_ps")
print("host  ", [getattr(bd, k) - float(g[k]) for k in keys])
eng = get_engine()
d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).to(eng.device)
for rep in range(2):
    e, fd = eng.evaluate(d(wl.system.pos), d(wl.system.charge), wl.box, wl.alpha, params.r_c, soe,
                         d(g["modes"]), _rb_commonv(float(g["H"]), P, wl.alpha), float(g["c_q"]))
    e = e.cpu().numpy()
    print("device", [e[i] - float(g[k]) for i, k in enumerate(keys)], "status", e[5])
u, fs = pk.short_range_energy_forces(wl.system, wl.box, wl.alpha, params.r_c)
print("short alone", u - float(g["u_s"]))
bd, f = pk.rb_energy_forces(wl.system, wl.box, params, soe, StubSampler(g["modes"]), P,
                            H=float(g["H"]), c_q=float(g["c_q"]))
print("host again", [getattr(bd, k) - float(g[k]) for k in keys])
