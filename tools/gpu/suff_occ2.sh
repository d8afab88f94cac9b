#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/bench_configs.py --only cfg1,cfg3,cfg4,cfg5 --no-cpu --policy 0 > gpurun_out/cfg_occ2.log 2>&1; echo "cfg rc=$?"
python -c "
import json
for l in open('gpurun_out/cfg_occ2.log'):
    if l.startswith('{'):
        d=json.loads(l); print(d['config'], round(d['gpu_chain_steps_per_s']), 'ms/step %.4f'%d['gpu_ms_per_step'])
"
bash tools/gpu/ncu_cmd.sh suff_cfg5 gauss_kernel 3 python tools/bench_configs.py --only cfg5 --no-cpu --policy 0 --steps 2 --warmup 1
bash tools/gpu/ncu_cmd.sh suff_cfg3 gauss_kernel 3 python tools/bench_configs.py --only cfg3 --no-cpu --policy 0 --steps 2 --warmup 1
for C in cfg3 cfg5 cfg2; do timeout 600 python tools/phase_times.py --config $C > gpurun_out/phase_$C.log 2>&1; tail -1 gpurun_out/phase_$C.log; done
