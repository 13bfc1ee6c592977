#!/bin/bash
timeout -s KILL 300 python -m pytest tests/test_gpu_kernels.py tests/test_api_gpu.py -q -x > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt.log
timeout -s KILL 200 python scripts/probe_perf.py 12 > gpurun_out/probe.log 2>&1; cat gpurun_out/probe.log
for d in 0.45 0.2; do FGA_LIB=build/variants/libtrace.so FGA_TRACE_IT=6 timeout -s KILL 100 python scripts/trace_run.py $d gpurun_out/trace_$d.txt > /dev/null 2>&1; python scripts/trace_report.py gpurun_out/trace_$d.txt; done
