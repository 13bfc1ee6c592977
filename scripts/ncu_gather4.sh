#!/bin/bash
# gather4-vs-LDGSTS producers of the attention kernel (round-1 build knobs at 3cb3ba1, built by
# scripts/build_rev.sh into build/variants/<name>):
#   g4base   : 4 balanced cp.async producers (the shipped design)      build_rev.sh 3cb3ba1 g4base
#   g4elect  : balanced producers, tile::gather4 from one elected lane  ... -DFGA_TMA_ELECT=1
#   g4split0 : one cp.async producer warp per ring slot                 ... -DFGA_PROD_SPLIT=0
#   g4lane   : one producer warp per slot, K and V by per-lane gather4  ... -DFGA_PROD_SPLIT=0 -DFGA_TMA_GATHER=3
# A/B timing + one ncu capture each.
mkdir -p gpurun_out
V=${V:-g4base g4elect g4split0 g4lane}
libs=""; for v in $V; do libs="$libs build/variants/$v/lib$v.so"; done
timeout -s KILL 300 python scripts/ab_attn.py $libs > gpurun_out/g4_ab.log 2>&1
for v in $V; do
  timeout -s KILL 300 ncu --set full --clock-control none -k regex:fga_attn -s 4 -c 1 -o gpurun_out/prof_$v -f \
    python scripts/ab_attn.py build/variants/$v/lib$v.so > gpurun_out/ncu_$v.log 2>&1
  echo "$v ncu rc=$?"
done
