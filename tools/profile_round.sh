#!/bin/bash
# Round profile evidence (run on the GPU box from the repo root):
#   bash tools/profile_round.sh r01
# 1. a plain bench run (the numbers), 2. the ncu launch list of the same command
# (cold-cache, serialised: shares, not absolutes), 3. one `--set full` capture per
# top kernel on a cfg4 step.  Summarise afterwards here with
#   python tools/summarize_ncu.py <tag> gpurun_out/launches_<tag>.csv gpurun_out/prof_<tag>_*.ncu-rep
set -e
TAG=${1:-r01}
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
for k in fourier_sweep fourier_sweep_rem fourier_aggregate_mma fourier_carry_rewrite fourier_carry_compose \
         pair_list nbr_build zero_sweep zero_aggregate_lane zero_carry radix_onesweep; do
  ncu --set full --clock-control none --import-source on -k regex:${k}_kernel -s 2 -c 1 \
      -f -o gpurun_out/prof_${TAG}_${k} python tools/one_step.py cfg4 3 \
      > gpurun_out/ncu_${k}.log 2>&1 || echo "capture ${k} failed"
done
