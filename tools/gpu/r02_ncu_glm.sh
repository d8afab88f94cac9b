#!/bin/bash
# full ncu capture of glm_kernel<logistic,52> (full-wave sampling launch) under the bench command
mkdir -p gpurun_out
bash tools/gpu/ncu_cmd.sh r02_glm glm_kernel 4 python bench.py --no-cpu --no-e2e --steps 2 --warmup 1
