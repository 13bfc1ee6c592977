#!/bin/bash
# A/B timing of variant libraries: ./scripts/ab.sh name1 name2 ...
for v in base "$@"; do
  if [ "$v" = base ]; then lib=""; else lib="build/variants/lib$v.so"; fi
  echo "== $v"; FGA_LIB=$lib timeout -s KILL 120 python scripts/probe_perf.py 12 0.45 2>&1 | grep -E "sparse|dense\(own"
done
