#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_fixtures.py tests/test_armijo.py tests/test_gpu_parity.py -m gpu -q --timeout 1200 -x > gpurun_out/r3k_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r3k_tests.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r3k_bench_C5.json 2> gpurun_out/r3k_bench_C5.err; echo "bench rc=$?"; python tools/bench_brief.py gpurun_out/r3k_bench_C5.json
KG_DEV=1 KG_NO_PDL=1 timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r3k_bench_C5_nopdl.json 2> gpurun_out/r3k_bench_C5_nopdl.err; echo "bench rc=$?"; python tools/bench_brief.py gpurun_out/r3k_bench_C5_nopdl.json
timeout 300 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r3k_bench_C3.json 2> gpurun_out/r3k_bench_C3.err; echo "C3 rc=$?"; python tools/bench_brief.py gpurun_out/r3k_bench_C3.json
