#!/bin/bash
# launch list + one --set full capture of the headline kernel with the current build (bench command)
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e"
timeout 300 $CMD > gpurun_out/plain.log 2>&1; echo "plain rc=$?"; tail -1 gpurun_out/plain.log | cut -c1-200
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v12.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:glm_kernel -s 4 -c 1 -o /tmp/prof_glm_v12 $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
ncu -i /tmp/prof_glm_v12.ncu-rep --page raw --csv > gpurun_out/prof_glm_v12_raw.csv 2>/dev/null
ncu -i /tmp/prof_glm_v12.ncu-rep --page details > gpurun_out/prof_glm_v12_details.txt 2>/dev/null
ncu -i /tmp/prof_glm_v12.ncu-rep --page source --csv > gpurun_out/prof_glm_v12_src.csv 2>/dev/null
ls -la gpurun_out | tail -4
