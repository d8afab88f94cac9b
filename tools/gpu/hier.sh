#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "radon or ex1 or grouped" > gpurun_out/pytest_hier.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_hier.log
timeout 600 python tools/bench_configs.py --only cfg3,cfg1 --no-cpu > gpurun_out/cfg_hier.log 2>&1; echo "cfg rc=$?"; cut -c1-330 gpurun_out/cfg_hier.log
timeout 600 python tools/bench_configs.py --only cfg3 --no-cpu --policy 1 >> gpurun_out/cfg_hier.log 2>&1; tail -1 gpurun_out/cfg_hier.log | cut -c1-330
