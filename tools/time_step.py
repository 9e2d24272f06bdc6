"""Quick CUDA-event timing of one device-resident evaluation per workload (dev tool)."""

import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2403_01521_b200 as pk  # noqa: E402
from paper_2403_01521_b200.configs import make_workload  # noqa: E402
from paper_2403_01521_b200.engine import DeviceEvaluator  # noqa: E402


def main(names, steps=5, graph=False):
    for name in names:
        t0 = time.time()
        wl = make_workload(name)
        soe = pk.build_soe_contour(wl.m)
        params = wl.params()
        ev = DeviceEvaluator(wl.system, wl.box, params, soe, P=wl.P, seed=wl.seed)
        ev.step()
        torch.cuda.synchronize()
        if graph:
            ev.capture()
        for _ in range(2):
            ev.step()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(steps):
            ev.step()
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / steps
        en = ev.energy.cpu().numpy()
        print(f"{name}: N={wl.n} P={ev.P} M={wl.m} {ms:.3f} ms/step  "
              f"{wl.n / ms * 1e3:.3e} particle-steps/s  E={en[:5]} status={en[5]} "
              f"(setup {time.time() - t0:.1f}s)", flush=True)


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    main(args or ["cfg1", "cfg2", "cfg3", "cfg4"], graph="--graph" in sys.argv)
