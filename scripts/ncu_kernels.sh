#!/bin/bash
# ncu launch list (fga kernels only) of a python script: ./scripts/ncu_kernels.sh script.py [args]
ncu --metrics gpu__time_duration.sum --clock-control none --csv python "$@" 2>/dev/null | grep -v "^==" > /tmp/ncu_k.csv
python - <<PY
import csv
rows=list(csv.reader(open("/tmp/ncu_k.csv")))
h=rows[0]
for r in rows[1:]:
    if len(r)==len(h) and ("fga" in r[h.index("Kernel Name")] or "unnamed" in r[h.index("Kernel Name")]): print(r[h.index("Kernel Name")][:60], r[h.index("Metric Value")])
PY
