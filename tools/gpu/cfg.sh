#!/bin/bash
# usage: bash tools/gpu/cfg.sh <configs> [policy]
mkdir -p gpurun_out
timeout 900 python tools/bench_configs.py --only $1 --no-cpu --policy ${2:-0} > gpurun_out/cfg.log 2>&1; echo "cfg rc=$?"
python -c "
import json
for l in open('gpurun_out/cfg.log'):
    if l.startswith('{'):
        d=json.loads(l); print(d['config'], d['policy'], round(d['gpu_chain_steps_per_s']), 'ms/step %.3f'%d['gpu_ms_per_step'], 'frac %.4f'%d['frac'])
    else: print(l.rstrip()[:200])
"
