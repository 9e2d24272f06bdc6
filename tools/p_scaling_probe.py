import sys
sys.path.insert(0, ".")
import torch
import paper_2403_01521_b200 as pk
from paper_2403_01521_b200.configs import make_workload
from paper_2403_01521_b200.engine import DeviceEvaluator
from torch.profiler import ProfilerActivity, profile
wl = make_workload("cfg4")
soe = pk.build_soe_contour(wl.m)
for P in (96, 100, 112, 128):
    ev = DeviceEvaluator(wl.system, wl.box, wl.params(), soe, P=P, seed=4)
    ev.warmup(); ev.step(); torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(3): ev.step()
        torch.cuda.synchronize()
    t = {e.key: e.device_time_total / 3e3 for e in prof.key_averages() if "fourier_sweep" in e.key or "aggregate_mma" in e.key}
    print(P, {k.split("(")[0][-40:]: round(v, 3) for k, v in t.items()})
    del ev
