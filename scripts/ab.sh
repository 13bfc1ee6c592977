#!/bin/bash
# A/B timing of variant libraries: ./scripts/ab.sh name1 name2 ...   (DENS env: densities)
for v in base "$@"; do
  if [ "$v" = base ]; then lib=""; else lib="build/variants/lib$v.so"; fi
  for d in ${DENS:-0.45}; do
    echo "== $v d=$d $(FGA_LIB=$lib timeout -s KILL 120 python scripts/probe_perf.py 12 $d 2>&1 | grep -E 'sparse')"
  done
done
