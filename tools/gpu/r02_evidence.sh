#!/bin/bash
# Round-2 evidence on one B200: GPU suite, smoke, bench (ours, reference arm, FP32), per-config table,
# ncu launch list of the bench command and full captures of the dominant kernels.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/ev_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/ev_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/ev_smoke.log
timeout 900 python bench.py > gpurun_out/ev_bench.log 2>&1; echo "bench rc=$?"; cut -c1-300 gpurun_out/ev_bench.log | grep -v "^glm_kernel"
timeout 900 python bench.py --impl reference > gpurun_out/ev_bench_ref.log 2>&1; echo "ref rc=$?"; cut -c1-300 gpurun_out/ev_bench_ref.log
timeout 600 python bench.py --fp32 > gpurun_out/ev_bench_fp32.log 2>&1; echo "fp32 rc=$?"; cut -c1-200 gpurun_out/ev_bench_fp32.log
timeout 1800 python tools/bench_configs.py > gpurun_out/ev_configs.jsonl 2>&1; echo "configs rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev_launches.csv python bench.py --no-cpu --no-e2e --steps 2 --warmup 1 > gpurun_out/ev_ncu_launches.log 2>&1; echo "launches rc=$?"
bash tools/gpu/ncu_cmd.sh ev_glm glm_kernel 4 python bench.py --no-cpu --no-e2e --steps 2 --warmup 1
bash tools/gpu/ncu_cmd.sh ev_lean_cfg5 lean_kernel 2 python tools/bench_configs.py --only cfg5 --no-cpu --policy 0 --steps 2 --warmup 1
bash tools/gpu/ncu_cmd.sh ev_lean_cfg1 lean_kernel 2 python tools/bench_configs.py --only cfg1 --no-cpu --policy 0 --steps 2 --warmup 1
bash tools/gpu/ncu_cmd.sh ev_lean_cfg4 lean_kernel 2 python tools/bench_configs.py --only cfg4 --no-cpu --policy 0 --steps 2 --warmup 1
