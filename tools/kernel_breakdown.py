"""Per-kernel device-time breakdown of one evaluation via torch.profiler (CUPTI)."""

import sys

import torch

sys.path.insert(0, ".")
import paper_2403_01521_b200 as pk  # noqa: E402
from paper_2403_01521_b200.configs import make_workload  # noqa: E402
from paper_2403_01521_b200.engine import DeviceEvaluator  # noqa: E402


def main(name, steps=2):
    wl = make_workload(name)
    soe = pk.build_soe_contour(wl.m)
    ev = DeviceEvaluator(wl.system, wl.box, wl.params(), soe, P=wl.P, seed=wl.seed)
    for _ in range(2):
        ev.step()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(steps):
            ev.step()
        torch.cuda.synchronize()
    rows = []
    for evt in prof.key_averages():
        t = getattr(evt, "device_time_total", None) or getattr(evt, "cuda_time_total", 0)
        if t > 0:
            rows.append((t / steps, evt.count // steps, evt.key))
    rows.sort(reverse=True)
    tot = sum(r[0] for r in rows)
    print(f"== {name}: N={wl.n} P={ev.P}  total device {tot / 1e3:.3f} ms/step")
    for t, c, k in rows[:25]:
        print(f"  {t / 1e3:9.3f} ms {100 * t / tot:5.1f}%  x{c:<4d} {k[:110]}")


if __name__ == "__main__":
    for n in sys.argv[1:] or ["cfg2", "cfg4"]:
        main(n)
