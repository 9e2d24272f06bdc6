"""Kernel timeline of one device-resident evaluation (torch.profiler / CUPTI):
start / end of every kernel relative to the step's first kernel, its stream,
and the idle gaps on the union of streams -- what sits on the critical path.

    python tools/timeline.py [config] [W rank]

With W and rank: that rank's share of a W-way sharded evaluation
(SHARD_MODE=modes|zsplit, the collectives skipped -- one GPU).
"""
import json
import os
import sys
import tempfile

import torch

sys.path.insert(0, ".")
import paper_2403_01521_b200 as pk  # noqa: E402
from paper_2403_01521_b200.configs import make_workload  # noqa: E402
from paper_2403_01521_b200.engine import DeviceEvaluator  # noqa: E402


def main(name="cfg4", W=1, rank=0):
    wl = make_workload(name)
    soe = pk.build_soe_contour(wl.m)
    if W > 1:
        ev = DeviceEvaluator(wl.system, wl.box, wl.params(), soe, P=wl.P, seed=wl.seed,
                             rank=rank, world=W,
                             shard_mode=os.environ.get("SHARD_MODE", "modes"))
        ev.reduce = False
        ev.exchange = lambda local, gathered: None
        ev.warmup()
    else:
        ev = DeviceEvaluator(wl.system, wl.box, wl.params(), soe, P=wl.P, seed=wl.seed)
    for _ in range(3):
        ev.step()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        ev.step()
        torch.cuda.synchronize()
    path = os.path.join(tempfile.mkdtemp(), "trace.json")
    prof.export_chrome_trace(path)
    evs = [e for e in json.load(open(path))["traceEvents"]
           if e.get("cat") == "kernel" and "dur" in e]
    evs.sort(key=lambda e: e["ts"])
    t0 = evs[0]["ts"]
    end = 0.0
    busy = []
    for e in evs:
        s, d = e["ts"] - t0, e["dur"]
        name_ = e["name"].replace("void slab::", "").replace("slab::", "").split("(")[0]
        print(f"{s / 1e3:8.3f} {(s + d) / 1e3:8.3f} ms  s{e['args'].get('stream', '?'):<4} {name_[:60]}")
        busy.append((s, s + d))
        end = max(end, s + d)
    # idle time on the union of streams
    busy.sort()
    idle, cur = 0.0, 0.0
    for s, t in busy:
        if s > cur:
            idle += s - cur
        cur = max(cur, t)
    print(f"span {end / 1e3:.3f} ms, idle gaps {idle / 1e3:.3f} ms")


if __name__ == "__main__":
    a = sys.argv[1:]
    main(a[0] if a else "cfg4", int(a[1]) if len(a) > 1 else 1, int(a[2]) if len(a) > 2 else 0)
