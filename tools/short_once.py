"""One device short-range evaluation of a workload (profiling target)."""
import sys
sys.path.insert(0, ".")
import paper_2403_01521_b200 as pk
from paper_2403_01521_b200.configs import make_workload

wl = make_workload(sys.argv[1] if len(sys.argv) > 1 else "cfg4")
for _ in range(2):
    u, f = pk.short_range_energy_forces(wl.system, wl.box, wl.alpha, wl.params().r_c)
print("u_s", u)
