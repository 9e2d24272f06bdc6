#!/bin/bash
# Round evidence, run on the GPU box from the repo root:
#   gpurun -- 'bash tools/round_evidence.sh r02'
# GPU suite, bench line, ncu launch list + full captures (summarised here into
# the profiles/ tables, then copied to gpurun_out/ev/ with only the two largest
# kernels' reports kept: gpurun merges back at most 64 MiB), reference arm and
# the per-config bench lines.
TAG=${1:-r02}
mkdir -p gpurun_out/ev
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/ev/gputest_final.log 2>&1
echo "tests rc=$?"
bash tools/profile_round.sh $TAG > gpurun_out/ev/profile_round.log 2>&1
echo "profile rc=$?"
cp gpurun_out/bench_plain.log gpurun_out/ev/bench_plain.log
python tools/summarize_ncu.py $TAG gpurun_out/launches_$TAG.csv gpurun_out/prof_${TAG}_*.ncu-rep \
  > gpurun_out/ev/summarize.log 2>&1
cp profiles/ncu_${TAG}_launches.md profiles/ncu_${TAG}_summary.json profiles/ncu_${TAG}_kernels.md \
  gpurun_out/launches_$TAG.csv gpurun_out/ev/ 2>/dev/null
for f in gpurun_out/prof_${TAG}_*.ncu-rep; do
  case $f in *fourier_sweep.ncu-rep|*pair_list.ncu-rep) mv $f gpurun_out/ev/ ;; *) rm -f $f ;; esac
done
rm -f gpurun_out/launches_$TAG.csv
timeout 900 python bench.py --impl reference > gpurun_out/ev/bench_reference.log 2>&1
echo "ref rc=$?"
for c in cfg1 cfg2 cfg3 cfg4 cfg5_1e4 cfg5_1e5 cfg5_1e6 cfg5_1e7; do
  timeout 600 python bench.py --config $c --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/ev/bc_$c.json
done
du -sh gpurun_out
echo done
