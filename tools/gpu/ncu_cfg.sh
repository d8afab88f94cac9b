#!/bin/bash
# usage: bash tools/gpu/ncu_cfg.sh <cfg> <kernel regex> <skip launches> <out name>
mkdir -p gpurun_out
CMD="python tools/bench_configs.py --only $1 --no-cpu --steps 2 --warmup 1"
timeout 600 $CMD > gpurun_out/plain_$4.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 -o gpurun_out/$4 $CMD > gpurun_out/ncu_$4.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/ncu_$4.log
