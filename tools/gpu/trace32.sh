#!/bin/bash
# Timeline of the FP32 kernel's control thread and epilogue warp 0 (CTA 0, pass 6): rebuilds the
# box's copy of libpcvg with -DPCVG_GLM32_TRACE and runs one short sampling call.
mkdir -p gpurun_out
PCVG_NVCC_DEFS=-DPCVG_GLM32_TRACE python -c "from paper_2310_07002_b200 import build; build.build(force=True)" || exit 1
timeout 300 python bench.py --fp32 --folds 2368 --steps 1 --warmup 3 > gpurun_out/trace32.log 2>&1
echo rc=$?; grep -A41 "^tile:" gpurun_out/trace32.log | head -45
