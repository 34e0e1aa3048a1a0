#!/bin/bash
# k_slab2 (scatter/gather Y) vs k_slab (DMMA Y): parity on the slab-route tests, kernel time, C5 bench
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "slab or poisson" --timeout 600 > gpurun_out/r3a_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r3a_tests.log
for c in C3 C5; do
  timeout 300 python tools/time_kernel.py --config $c --which 0 --reps 20
  KG_DEV=1 KG_SLAB_DMMA=1 timeout 300 python tools/time_kernel.py --config $c --which 0 --reps 20
done
timeout 900 python -m pytest tests/test_gpu_fixtures.py -m gpu -q --timeout 800 > gpurun_out/r3a_fixtures.log 2>&1; echo "fixtures rc=$?"; tail -3 gpurun_out/r3a_fixtures.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r3a_bench_C5.json 2> gpurun_out/r3a_bench_C5.err; echo "bench rc=$?"; cat gpurun_out/r3a_bench_C5.json
