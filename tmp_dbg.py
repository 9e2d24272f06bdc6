import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2403_01521_b200 as pk
from helpers import StubSampler, load_golden
from paper_2403_01521_b200.configs import make_workload
g = load_golden("cfg1"); wl = make_workload("cfg1")
soe = pk.build_soe_contour(wl.m); params = wl.params()
print("P", int(g["P"]), "nmodes", params.kmodes.shape)
for it in range(3):
    bd, f = pk.soe_energy_forces(wl.system, wl.box, params, soe)
    err = np.abs(f - g["forces"]).max(axis=1) / float(g["fmax"])
    bad = np.where(err > 1e-9)[0]
    print(it, bd.total, float(g["total"]), "bad", len(bad), bad[:8], f[bad[:2]], g["forces"][bad[:2]])
