#!/bin/bash
# Round-1 evidence after the sufficient-statistics kernel: GPU suite, smoke, bench (default +
# reference arm), per-config table with the CPU reference leg (AUTO and ROWS), convergence runs.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | cut -c1-200
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref.log | cut -c1-200
timeout 1500 python tools/bench_configs.py --policy 0 > gpurun_out/cfg_auto.log 2>&1; echo "cfg auto rc=$?"
timeout 600 python bench.py --fp32 --no-cpu > gpurun_out/bench_fp32.log 2>&1; echo "fp32 rc=$?"
timeout 900 python tools/bench_configs.py --policy 5 --no-cpu > gpurun_out/cfg_rows.log 2>&1; echo "cfg rows rc=$?"
for C in cfg1 cfg2 cfg3 cfg4 cfg5; do
  timeout 900 python tools/converge.py --config $C --fit > gpurun_out/conv_$C.log 2>&1; echo "conv $C rc=$?"
done
