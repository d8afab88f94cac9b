#!/bin/bash
# glm kernel (cfg2): logistic parity + bench line (device-timed only) + the K-fold / few-chain row
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bench_shapes.py tests/test_gpu_parity.py tests/test_gpu_edge.py -q -m gpu -x -k "cfg2 or logistic or tail or cluster" > gpurun_out/r02_glm_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02_glm_pytest.log
timeout 900 python bench.py --no-cpu --no-e2e --steps 10 --warmup 3 > gpurun_out/r02_glm_bench.log 2>&1; echo "bench rc=$?"; cut -c1-400 gpurun_out/r02_glm_bench.log
timeout 600 python tools/bench_configs.py --only cfg2k,cfg1 --no-cpu --policy 2 > gpurun_out/r02_glm_cfg.log 2>&1; cut -c1-300 gpurun_out/r02_glm_cfg.log
