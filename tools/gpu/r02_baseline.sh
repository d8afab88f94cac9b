#!/bin/bash
# Round-2 baseline: per-config rates (AUTO policy), time-to-converged under the D_min early-stop
# rule, and full ncu captures of the sufficient-statistics kernel on cfg5 / cfg1 / cfg4.
mkdir -p gpurun_out
timeout 900 python tools/bench_configs.py --only cfg1,cfg3,cfg4,cfg5,cfg2,cfg2k --no-cpu --policy 0 > gpurun_out/r02_cfg_base.log 2>&1; echo "cfg rc=$?"
for C in cfg1 cfg3 cfg4 cfg5; do timeout 600 python tools/converge.py --config $C --no-cpu > gpurun_out/r02_conv_$C.log 2>&1; tail -1 gpurun_out/r02_conv_$C.log | cut -c1-600; done
bash tools/gpu/ncu_cmd.sh r02_suff_cfg5 gauss_kernel 3 python tools/bench_configs.py --only cfg5 --no-cpu --policy 0 --steps 2 --warmup 1
bash tools/gpu/ncu_cmd.sh r02_suff_cfg1 gauss_kernel 3 python tools/bench_configs.py --only cfg1 --no-cpu --policy 0 --steps 2 --warmup 1
bash tools/gpu/ncu_cmd.sh r02_suff_cfg4 gauss_kernel 3 python tools/bench_configs.py --only cfg4 --no-cpu --policy 0 --steps 2 --warmup 1
