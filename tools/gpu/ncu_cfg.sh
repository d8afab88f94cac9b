#!/bin/bash
# usage: bash tools/gpu/ncu_cfg.sh <cfg> <kernel regex> <skip launches> <out name> [keep]
# Full ncu capture of one launch; the raw + source pages are exported as CSV on the box (the
# .ncu-rep is kept only with a 5th argument, it can exceed gpurun's 64 MiB copy-back limit).
mkdir -p gpurun_out
CMD="python tools/bench_configs.py --only $1 --no-cpu --steps 2 --warmup 1"
timeout 600 $CMD > gpurun_out/plain_$4.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 -o /tmp/$4 $CMD > gpurun_out/ncu_$4.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/ncu_$4.log
ncu -i /tmp/$4.ncu-rep --page raw --csv > gpurun_out/$4_raw.csv 2>/dev/null
ncu -i /tmp/$4.ncu-rep --page source --csv > gpurun_out/$4_src.csv 2>/dev/null
ncu -i /tmp/$4.ncu-rep --page details > gpurun_out/$4_details.txt 2>/dev/null
if [ -n "$5" ]; then cp /tmp/$4.ncu-rep gpurun_out/; fi
ls -la gpurun_out | tail -5
