#!/bin/bash
# Round-1 evidence: full GPU suite, smoke, bench (default), launch list + ncu --set full of the
# headline kernel (glm_kernel<3,52>) and of the cfg3 batched kernel; CSV exports only.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; cat gpurun_out/smoke.log | tail -1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | cut -c1-300
CMD="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v5.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:glm_kernel -s 4 -c 1 -o /tmp/prof_glm_v5 $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
ncu -i /tmp/prof_glm_v5.ncu-rep --page raw --csv > gpurun_out/prof_glm_v5_raw.csv 2>/dev/null
ncu -i /tmp/prof_glm_v5.ncu-rep --page details > gpurun_out/prof_glm_v5_details.txt 2>/dev/null
bash tools/gpu/ncu_cfg.sh cfg3 gauss_kernel 3 prof_cfg3_v3
