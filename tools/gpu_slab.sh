#!/bin/bash
# slab-route check: kernel timings (slab pass + mode-3 steps), C5/C3 path wall times, fixture parity
mkdir -p gpurun_out
(timeout 300 python tools/time_kernel.py --config C5 --which 0 6 7; timeout 300 python tools/time_kernel.py --config C3 --which 0 6 7) > gpurun_out/slab_tk.log 2>&1; echo "tk rc=$?"; cat gpurun_out/slab_tk.log | tail -8
(timeout 300 python tools/prof_path.py --config C5 --paths 2; timeout 300 python tools/prof_path.py --config C3 --paths 2) > gpurun_out/slab_path.log 2>&1; echo "path rc=$?"; cat gpurun_out/slab_path.log | tail -5
timeout 900 python -m pytest tests/test_gpu_fixtures.py tests/test_gpu_parity.py tests/test_armijo.py -q --timeout 600 > gpurun_out/slab_tests.log 2>&1; echo "tests rc=$?"; grep -E "^FAILED|^E  |passed|failed" gpurun_out/slab_tests.log | head -30
