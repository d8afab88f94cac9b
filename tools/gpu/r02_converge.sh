#!/bin/bash
# time to R-hat-converged elpd under the sound early-stop rule (GPU, all configs) + the reference for cfg1
mkdir -p gpurun_out
for C in cfg1 cfg3 cfg4 cfg5; do timeout 900 python tools/converge.py --config $C --iters 2000 --fit > gpurun_out/r02_converge_$C.log 2>&1; tail -1 gpurun_out/r02_converge_$C.log | cut -c1-400; done
timeout 900 python tools/converge_ref.py --config cfg1 > gpurun_out/r02_converge_ref_cfg1.log 2>&1; tail -1 gpurun_out/r02_converge_ref_cfg1.log | cut -c1-400
timeout 1500 python tools/converge.py --config cfg2 --iters 1000 --no-cpu > gpurun_out/r02_converge_cfg2.log 2>&1; tail -1 gpurun_out/r02_converge_cfg2.log | cut -c1-400
