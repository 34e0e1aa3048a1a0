#!/bin/bash
# GPU-box recipe: test suite, then one full ncu capture each of the C2
# whole-path kernel and the C2 fused n-space pass (kg_time_kernel), written to
# gpurun_out/ for summarising under profiles/.
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/gpu_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests.log
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_gauss_path -c 1 \
  -o gpurun_out/r01_c2_path python tools/prof_path.py --config C2 --paths 1 > gpurun_out/ncu_path.log 2>&1
echo "ncu path rc=$?"
timeout 300 ncu --set full --clock-control none -k regex:k_fused_fast -c 1 -s 2 \
  -o gpurun_out/r01_c2_fused python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_fused.log 2>&1
echo "ncu fused rc=$?"
