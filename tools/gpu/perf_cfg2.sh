#!/bin/bash
# quick cfg2 check: gpu parity tests of the glm kernel + bench (no cpu leg) + probes
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "logistic or tensor" > gpurun_out/pytest_glm.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_glm.log
timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/bench_quick.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_quick.log | cut -c1-400
if [ "$1" == "probe" ]; then
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dmma_latency tools/probes/dmma_latency.cu && timeout 120 /tmp/dmma_latency > gpurun_out/dmma_latency.log 2>&1; cat gpurun_out/dmma_latency.log
fi
