#!/bin/bash
# A/B of the in-tree library against _variants/<name>.so: graph step time (alternated) + kernel breakdown
for r in 1 2; do
  for v in "" "$@"; do
    if [ -z "$v" ]; then echo "== new"; python tools/time_step.py --graph ${CFG:-cfg4} 2>&1 | grep ms/step;
    else echo "== $v"; SLAB_B200_LIB=_variants/$v.so python tools/time_step.py --graph ${CFG:-cfg4} 2>&1 | grep ms/step; fi
  done
done
TOP=${TOP:-14} bash tools/ab_kernels.sh "$@"
