#!/bin/bash
# lean kernel: parity (engine / parity suites on the affected fixtures) and per-config rates
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_bench_shapes.py tests/test_gpu_parity.py -q -m gpu -x -k "lean or short_horizon or within_mcse or cfg1 or seasonal or bench_shape" > gpurun_out/r02_lean_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r02_lean_pytest.log
for V in "PCVG_NO_LEAN=1" "PCVG_LEAN_MINB=1" "PCVG_LEAN_MINB=3" "PCVG_LEAN_MINB=4"; do
  env $V timeout 900 python tools/bench_configs.py --only cfg1,cfg4,cfg5 --no-cpu --policy 0 > gpurun_out/r02_lean_cfg_$V.log 2>&1
  python -c "
import json,sys
for l in open('gpurun_out/r02_lean_cfg_$V.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$V', d['config'], round(d['gpu_chain_steps_per_s']), 'ms/step %.4f'%d['gpu_ms_per_step'], d['elpd_sum_model0'])
"
done
