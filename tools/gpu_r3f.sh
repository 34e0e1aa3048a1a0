#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "slab_route or poisson" --timeout 600 > gpurun_out/r3f_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r3f_tests.log
timeout 300 python tools/time_kernel.py --config C5 --which 0 --reps 20
timeout 300 python tools/time_kernel.py --config C3 --which 0 --reps 20
