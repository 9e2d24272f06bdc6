"""Run a workload's device step a few times (for ncu / compute-sanitizer targets)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2403_01521_b200 as pk  # noqa: E402
from paper_2403_01521_b200.configs import make_workload  # noqa: E402
from paper_2403_01521_b200.engine import DeviceEvaluator  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
wl = make_workload(name)
soe = pk.build_soe_contour(wl.m)
ev = DeviceEvaluator(wl.system, wl.box, wl.params(), soe, P=wl.P, seed=wl.seed)
for _ in range(steps):
    ev.step()
torch.cuda.synchronize()
print(name, ev.energy.cpu().numpy()[:6])
