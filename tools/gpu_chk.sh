#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fixtures.py -m gpu -q --timeout 1200 -x > gpurun_out/r3m_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r3m_tests.log
timeout 300 python tools/time_kernel.py --config C5 --which 0 --reps 20
timeout 300 python tools/time_kernel.py --config C3 --which 0 --reps 20
