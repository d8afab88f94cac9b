#!/bin/bash
# lanes-per-chain sweep of the sufficient-statistics kernel + one ncu capture (cfg4, T=1)
mkdir -p gpurun_out
for T in 1 4 8 32; do
  PCVG_SUFF_LANES=$T timeout 600 python tools/bench_configs.py --only cfg1,cfg3,cfg4 --no-cpu --policy 4 > gpurun_out/lanes_$T.log 2>&1
  python -c "
import json
for l in open('gpurun_out/lanes_$T.log'):
    if l.startswith('{'):
        d=json.loads(l); print('T=$T', d['config'], round(d['gpu_chain_steps_per_s']), 'ms/step %.4f'%d['gpu_ms_per_step'])
"
done
export PCVG_SUFF_LANES=1
bash tools/gpu/ncu_cmd.sh suff_cfg4 gauss_kernel 6 python tools/bench_configs.py --only cfg4 --no-cpu --policy 4 --steps 2 --warmup 1
