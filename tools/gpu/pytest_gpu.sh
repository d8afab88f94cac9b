#!/bin/bash
# usage: bash tools/gpu/pytest_gpu.sh [pytest -k expression]
mkdir -p gpurun_out
if [ -n "$1" ]; then K=(-k "$1"); else K=(); fi
timeout 1500 python -m pytest tests -m gpu -q -x "${K[@]}" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"
tail -30 gpurun_out/pytest_gpu.log
