#!/bin/bash
# quick GPU iteration: parity subset + timeline trace + layer timing
timeout -s KILL 200 python -m pytest tests/test_gpu_kernels.py -q -x -k "golden or dense or group or single or lse" > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pt.log
timeout -s KILL 100 python scripts/trace_run.py ${1:-0.45} gpurun_out/trace.txt > gpurun_out/trace_run.log 2>&1
timeout -s KILL 200 python scripts/probe_perf.py 12 ${1:-0.45} > gpurun_out/probe.log 2>&1; cat gpurun_out/probe.log
