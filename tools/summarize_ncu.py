"""Summarise ncu outputs into profiles/ (committed evidence).

    python tools/summarize_ncu.py <round_tag> <launches.csv> <full.ncu-rep> [more.ncu-rep ...]

Writes profiles/ncu_<tag>_launches.md (per-kernel share of one step from the
cold-cache serialised launch list) and profiles/ncu_<tag>_summary.json (per-kernel
metrics of the `--set full` capture: duration, DRAM bytes, fp64 pipe, IPC, ...).
"""

import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCAN = ("fourier_aggregate", "fourier_carry", "fourier_sweep", "zero_aggregate", "zero_carry",
        "zero_sweep", "decay_table", "chunk_bounds", "mode_table", "zero_chunk_decay")


def short(name):
    name = name.split("(")[0].replace("void ", "").replace("slab::", "")
    return name


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[hdr_i + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        k = short(r[ki])
        tot[k] += float(r[vi].replace(",", ""))
        cnt[k] += 1
    return tot, cnt


def full_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    want = {
        "gpu__time_duration.sum": "duration",
        "dram__bytes_read.sum": "dram_read",
        "dram__bytes_write.sum": "dram_write",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_inst_pct",
        "smsp__inst_executed.sum": "warp_inst",
        "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
        "launch__registers_per_thread": "registers",
        "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
        "smsp__thread_inst_executed_per_inst_executed.ratio": "threads_per_inst",
        "launch__grid_size": "grid",
        "launch__block_size": "block",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active":
            "dmma_pipe_pct",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active": "shared_pipe_pct",
        "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1_pct",
        "l1tex__t_sector_pipe_lsu_mem_global_op_ld_hit_rate.pct": "l1_hit_pct",
        "launch__occupancy_limit_registers": "occ_limit_regs",
    }
    scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "usecond": 1e-3,
             "msecond": 1.0, "nsecond": 1e-6, "us": 1e-3, "ms": 1.0, "ns": 1e-6}
    res = []
    for r in data:
        d = {"kernel": short(r[hdr.index("Kernel Name")])}
        for k, nm in want.items():
            if k in hdr:
                i = hdr.index(k)
                v = r[i].replace(",", "")
                try:
                    v = float(v) * scale.get(units[i], 1.0)
                except ValueError:
                    pass
                d[nm] = v
        d["duration_ms"] = d.pop("duration", None)
        res.append(d)
    return res


def main():
    tag, lpath, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    tot, cnt = launches(lpath)
    # not part of the evaluation step: bench.py's live DFMA peak probe, torch fills
    extra = {k: tot.pop(k) for k in list(tot) if k.startswith("dfma_peak") or k.startswith("at::")}
    grand = sum(tot.values())
    lines = [f"# ncu launch list, round {tag}", "",
             "`ncu --metrics gpu__time_duration.sum --clock-control none` over "
             "`python bench.py --steps 2 --warmup 3 --no-cpu-baseline` (cold-cache, serialised "
             "launches: compare SHARES, not absolute times).", "",
             "| kernel | launches | total ms | share |", "|---|---:|---:|---:|"]
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        lines.append(f"| {k} | {cnt[k]} | {v / 1e6:.3f} | {100 * v / grand:.1f}% |")
    scan = sum(v for k, v in tot.items() if any(k.startswith(s) for s in SCAN))
    lines += ["", f"SOE-scan kernels (3-phase Fourier scan + k=0 mode + tables): "
              f"{100 * scan / grand:.1f}% of device time.", "",
              "Excluded (outside the evaluation step): " +
              ", ".join(f"{k} ({v / 1e6:.3f} ms)" for k, v in extra.items())]
    with open(os.path.join(REPO, "profiles", f"ncu_{tag}_launches.md"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    full = [d for rep in reps for d in full_metrics(rep)]
    per_kernel = defaultdict(list)
    for d in full:
        per_kernel[d["kernel"]].append(d)
    summary = {"round": tag, "source": [os.path.basename(r) for r in reps], "kernels": {}}
    scan_bytes = 0.0
    for k, ds in per_kernel.items():
        d = ds[-1]
        summary["kernels"][k] = d
        if any(k.startswith(s) for s in SCAN):
            scan_bytes += (d.get("dram_read") or 0) + (d.get("dram_write") or 0)
    summary["scan_dram_bytes_per_step"] = scan_bytes
    summary["note"] = ("one launch per kernel per step; dram bytes = dram__bytes_read.sum + "
                       "dram__bytes_write.sum from ncu --set full")
    with open(os.path.join(REPO, "profiles", f"ncu_{tag}_summary.json"), "w") as fh:
        json.dump(summary, fh, indent=1)
    # one markdown table of the per-kernel limiters (the numbers DESIGN.md cites)
    tbl = [f"# ncu full captures, round {tag}", "",
           "`ncu --set full --clock-control none --import-source on` of one launch per kernel "
           "on a cfg4 step (`tools/profile_round.sh`).  fp64 = DFMA pipe; DMMA = the FP64 "
           "tensor sub-pipe; shared = the pipe both issue to; L1 = l1tex throughput.", "",
           "| kernel | ms | fp64 % | DMMA % | shared % | issue % | L1 % | L1 hit % | occupancy % "
           "| regs | DRAM MB |", "|---|---:|---:|---:|---:|---:|---:|---:|---:|---:|---:|"]

    def f(d, k, fmt="{:.1f}"):
        v = d.get(k)
        return fmt.format(v) if isinstance(v, float) else "-"
    for k, d in sorted(summary["kernels"].items(), key=lambda kv: -(kv[1].get("duration_ms")
                                                                    or 0)):
        mb = ((d.get("dram_read") or 0) + (d.get("dram_write") or 0)) / 1e6
        tbl.append(f"| {k} | {f(d, 'duration_ms', '{:.3f}')} | {f(d, 'fp64_pipe_pct')} | "
                   f"{f(d, 'dmma_pipe_pct')} | {f(d, 'shared_pipe_pct')} | "
                   f"{f(d, 'issue_active_pct')} | {f(d, 'l1_pct')} | {f(d, 'l1_hit_pct')} | "
                   f"{f(d, 'occupancy_pct')} | {f(d, 'registers', '{:.0f}')} | {mb:.0f} |")
    with open(os.path.join(REPO, "profiles", f"ncu_{tag}_kernels.md"), "w") as fh:
        fh.write("\n".join(tbl) + "\n")
    print("\n".join(lines[-12:]))
    print(json.dumps(summary, indent=1)[:3000])


if __name__ == "__main__":
    main()
