#!/bin/bash
# suffstat kernel: parity tests + per-config rates (policy 4) next to the row kernels (policy 0)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "suffstat or ragged or poisoned" > gpurun_out/pytest_suff.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_suff.log
timeout 900 python tools/bench_configs.py --only cfg1,cfg3,cfg4,cfg5 --no-cpu --policy 4 > gpurun_out/cfg_suff.log 2>&1; echo "cfg rc=$?"
cut -c1-420 gpurun_out/cfg_suff.log
