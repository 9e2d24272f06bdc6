#!/usr/bin/env bash
# A/B: per-kernel device times of a cfg step for the in-tree library and each
# _variants/<name>.so given on the command line (built with `make variant`).
cfg=${CFG:-cfg4}
echo "== base"; python tools/kernel_breakdown.py $cfg 2>&1 | grep -v -i warn | head -${TOP:-6}
for v in "$@"; do
  echo "== $v"; SLAB_B200_LIB=_variants/$v.so python tools/kernel_breakdown.py $cfg 2>&1 | grep -v -i warn | head -${TOP:-6}
done
