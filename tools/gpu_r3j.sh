#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 1200 -k "slab" > gpurun_out/r3j_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r3j_tests.log
