#!/bin/bash
# ncu --set full capture of one attention launch (c2, density $1) + launch list of the bench command
D=${1:-0.45}
mkdir -p gpurun_out
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:fga_attn_ws -s 2 -c 1 \
  -o gpurun_out/prof_attn -f python bench.py --steps 1 --warmup 2 --no-extras --density $D > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"; tail -3 gpurun_out/ncu_full.log
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-extras --density $D > gpurun_out/ncu_launch.log 2>&1
echo "ncu launches rc=$?"
