#!/bin/bash
# one-lane suff kernel with the 4-CTA/SM register bound: rates on cfg1/cfg4/cfg5 + gpu parity subset
mkdir -p gpurun_out
timeout 900 python tools/bench_configs.py --only cfg1,cfg3,cfg4,cfg5 --no-cpu --policy 0 > gpurun_out/cfg_occ.log 2>&1; echo "cfg rc=$?"
python -c "
import json
for l in open('gpurun_out/cfg_occ.log'):
    if l.startswith('{'):
        d=json.loads(l); print(d['config'], round(d['gpu_chain_steps_per_s']), 'ms/step %.4f'%d['gpu_ms_per_step'])
"
timeout 1200 python -m pytest tests -m gpu -q -x -k "suffstat or adapt or edge" > gpurun_out/pytest_occ.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_occ.log
