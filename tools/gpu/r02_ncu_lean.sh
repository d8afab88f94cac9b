#!/bin/bash
# ncu --set full of the lean kernel on cfg5 (many chains) and cfg1 (few chains)
mkdir -p gpurun_out
bash tools/gpu/ncu_cmd.sh r02_lean_cfg5 lean_kernel 2 python tools/bench_configs.py --only cfg5 --no-cpu --policy 0 --steps 2 --warmup 1
bash tools/gpu/ncu_cmd.sh r02_lean_cfg1 lean_kernel 2 python tools/bench_configs.py --only cfg1 --no-cpu --policy 0 --steps 2 --warmup 1
