#!/bin/bash
# full GPU suite with AUTO = sufficient statistics; per-config rates (auto vs row kernels);
# wall-clock to converged elpd per config
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
for P in 0 5; do
  timeout 900 python tools/bench_configs.py --only cfg1,cfg3,cfg4,cfg5 --no-cpu --policy $P > gpurun_out/cfg_p$P.log 2>&1; echo "cfg p$P rc=$?"
  python -c "
import json
for l in open('gpurun_out/cfg_p$P.log'):
    if l.startswith('{'):
        d=json.loads(l); print('policy $P', d['config'], round(d['gpu_chain_steps_per_s']), 'ms/step %.4f'%d['gpu_ms_per_step'])
"
done
for C in cfg1 cfg3 cfg4 cfg5; do
  timeout 900 python tools/converge.py --config $C --no-cpu > gpurun_out/conv_$C.log 2>&1; echo "conv $C rc=$?"; tail -1 gpurun_out/conv_$C.log | cut -c1-400
done
