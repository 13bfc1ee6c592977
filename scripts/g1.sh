#!/bin/bash
./scripts/gather_bench2 0.45 > gpurun_out/gb2_045.log 2>&1; cat gpurun_out/gb2_045.log
./scripts/gather_bench2 0.2 > gpurun_out/gb2_020.log 2>&1; cat gpurun_out/gb2_020.log
for d in 0.45 0.2; do FGA_TRACE_IT=6 timeout -s KILL 100 python scripts/trace_run.py $d gpurun_out/trace_$d.txt 2>&1 | grep -v "^\[" ; done
