#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
timeout 900 python tools/bench_configs.py --only cfg1,cfg3,cfg4,cfg5 --no-cpu --policy 0 > gpurun_out/cfg_p0b.log 2>&1; echo "cfg rc=$?"
python -c "
import json
for l in open('gpurun_out/cfg_p0b.log'):
    if l.startswith('{'):
        d=json.loads(l); print(d['config'], round(d['gpu_chain_steps_per_s']), 'ms/step %.4f'%d['gpu_ms_per_step'])
"
