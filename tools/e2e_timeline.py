"""GPU timeline (kernels and copies) of one public-API rb_energy_forces call
with page-locked host arrays: where the end-to-end time beyond the device step
goes.

    python tools/e2e_timeline.py [config] [--pageable]
"""
import json
import os
import sys
import tempfile

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2403_01521_b200 as pk  # noqa: E402
from paper_2403_01521_b200 import rbse2d  # noqa: E402
from paper_2403_01521_b200.configs import make_workload  # noqa: E402
from paper_2403_01521_b200.engine import pinned_like  # noqa: E402


def main(name="cfg4"):
    wl = make_workload(name)
    soe = pk.build_soe_contour(wl.m)
    params = wl.params()
    H = rbse2d.normalization_H(wl.alpha, wl.box)
    c_q = rbse2d.charge_term_sum(wl.alpha, wl.box, float(np.sum(wl.system.charge ** 2)))
    s = pk.make_system(wl.system.charge, wl.system.mass, wl.system.pos, box=wl.box)
    if "--pageable" not in sys.argv:
        s.pos = pinned_like(wl.system.pos)
        s.charge = pinned_like(wl.system.charge)
    smp = rbse2d.ModeSampler(wl.alpha, wl.box, seed=wl.seed)
    for _ in range(3):
        pk.rb_energy_forces(s, wl.box, params, soe, smp, wl.P, H=H, c_q=c_q)
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        pk.rb_energy_forces(s, wl.box, params, soe, smp, wl.P, H=H, c_q=c_q)
        torch.cuda.synchronize()
    path = os.path.join(tempfile.mkdtemp(), "trace.json")
    prof.export_chrome_trace(path)
    evs = json.load(open(path))["traceEvents"]
    gpu = [e for e in evs if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "dur" in e]
    cpu = [e for e in evs if e.get("cat") == "cuda_runtime" and "dur" in e]
    allev = gpu + cpu
    t0 = min(e["ts"] for e in allev)
    gpu.sort(key=lambda e: e["ts"])
    end = max(e["ts"] + e["dur"] for e in gpu)
    print(f"first runtime call at 0, first GPU op at {(gpu[0]['ts'] - t0) / 1e3:.3f} ms, "
          f"last GPU op ends {(end - t0) / 1e3:.3f} ms")
    for e in gpu:
        if e["cat"] != "kernel" or e["dur"] > 30 or e["ts"] - t0 < 3000:
            nm = e["name"].replace("void slab::", "").split("(")[0][:50]
            print(f"{(e['ts'] - t0) / 1e3:8.3f} {(e['ts'] + e['dur'] - t0) / 1e3:8.3f}  "
                  f"{e['cat']:10s} s{e['args'].get('stream', '?'):<4} {nm}")
    for e in sorted(cpu, key=lambda e: e["ts"]):
        if e["ts"] - t0 < 2600 and e["dur"] > 20:
            print(f"cpu {e['name'][:40]:40s} {(e['ts'] - t0) / 1e3:8.3f} + {e['dur'] / 1e3:.3f} ms")
    syncs = [e for e in cpu if "Synchronize" in e["name"]]
    for e in syncs:
        print(f"sync {e['name']} {(e['ts'] - t0) / 1e3:.3f} + {e['dur'] / 1e3:.3f} ms")


if __name__ == "__main__":
    main(*([a for a in sys.argv[1:2] if not a.startswith("--")] or ["cfg4"]))
