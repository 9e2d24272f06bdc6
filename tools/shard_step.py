"""Device time of ONE rank's share of a sharded evaluation (rank r of W), on one GPU.

    python tools/shard_step.py [config] [W]

Times DeviceEvaluator(rank=0..W-1, world=W).step() with the all-reduce disabled for each rank
in turn, its local parts replayed as CUDA graphs like bench.py does (SHARD_GRAPH=0: eager) -- the per-GPU work of the multi-GPU run without the NCCL all-reduce
(the driver's scaling run measures the real thing)."""
import sys

import os

import torch

sys.path.insert(0, ".")
import paper_2403_01521_b200 as pk  # noqa: E402
from paper_2403_01521_b200.configs import make_workload  # noqa: E402
from paper_2403_01521_b200.engine import DeviceEvaluator  # noqa: E402

MODE = os.environ.get("SHARD_MODE", "zsplit")
GRAPH = os.environ.get("SHARD_GRAPH", "1") == "1"  # the rank's parts replayed as CUDA graphs


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
    W = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    wl = make_workload(name)
    soe = pk.build_soe_contour(wl.m)
    params = wl.params()
    for r in range(W):
        ev = DeviceEvaluator(wl.system, wl.box, params, soe, P=wl.P, seed=wl.seed, rank=r,
                             world=W, shard_mode=MODE)
        ev.reduce = False  # one GPU: time the rank's own work only
        ev.exchange = lambda local, gathered: None  # (results meaningless; timing only)
        ev.warmup()
        if GRAPH:
            ev.capture()
        for _ in range(2):
            ev.step()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(5):
            ev.step()
        e.record()
        torch.cuda.synchronize()
        print(f"{name} rank {r}/{W}: {s.elapsed_time(e) / 5:.3f} ms/step")
        del ev




def profile_rank(name="cfg4", W=8, r=1):
    from torch.profiler import ProfilerActivity, profile
    wl = make_workload(name)
    soe = pk.build_soe_contour(wl.m)
    ev = DeviceEvaluator(wl.system, wl.box, wl.params(), soe, P=wl.P, seed=wl.seed, rank=r,
                         world=W, shard_mode=MODE)
    ev.reduce = False
    ev.exchange = lambda local, gathered: None
    ev.warmup()
    ev.step()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(3):
            ev.step()
        torch.cuda.synchronize()
    rows = sorted(((e.device_time_total / 1e3 / 3, e.key) for e in prof.key_averages()
                   if e.device_time_total > 0), reverse=True)
    print(f"  total device {sum(r[0] for r in rows):.3f} ms/step")
    for ms, k in rows[:16]:
        print(f"  {ms:8.3f} ms/step  {k[:90]}")


if __name__ == "__main__":
    if len(sys.argv) > 3 and sys.argv[3] == "profile":
        profile_rank(sys.argv[1], int(sys.argv[2]))
    else:
        main()
