"""Debug: device short range at a golden config against the reference's sampled forces."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2403_01521_b200 as pk
from paper_2403_01521_b200.configs import make_workload

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5_1e7"
g = dict(np.load(f"tests/golden/{name}.npz"))
wl = make_workload(name)
u, f = pk.short_range_energy_forces(wl.system, wl.box, wl.alpha, wl.params().r_c)
print(name, "u_s", repr(u), "ref", repr(float(g["u_s_alone"])), "diff", u - float(g["u_s_alone"]))
idx = g["sample_idx"] if "sample_idx" in g else np.arange(wl.n)
d = np.max(np.abs(f[idx] - g["f_short"]), axis=1)
bad = np.argsort(d)[::-1][:8]
L = np.array([wl.box.lx, wl.box.ly, wl.box.lz])
print("max force err", d.max(), "n bad(>1e-9)", int((d > 1e-9).sum()), "of", len(idx))
for b in bad:
    i = idx[b]
    print(i, d[b], wl.system.pos[i], wl.system.pos[i] / L)
