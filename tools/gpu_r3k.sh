#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_fixtures.py tests/test_armijo.py -m gpu -q --timeout 1200 > gpurun_out/r3k_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r3k_tests.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r3k_bench_C5.json 2> gpurun_out/r3k_bench_C5.err; echo "bench rc=$?"; python -c "import json; d=json.load(open('gpurun_out/r3k_bench_C5.json')); print('fork', d['ms_per_step'], d['value'], d['e2e']['ms_per_step'], d['gpu_launches'])"
KG_DEV=1 KG_NO_FORK=1 timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r3k_bench_C5_nofork.json 2> gpurun_out/r3k_bench_C5_nofork.err; echo "bench rc=$?"; python -c "import json; d=json.load(open('gpurun_out/r3k_bench_C5_nofork.json')); print('nofork', d['ms_per_step'], d['value'], d['e2e']['ms_per_step'])"
timeout 300 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r3k_bench_C3.json 2> gpurun_out/r3k_bench_C3.err; echo "C3 rc=$?"; python -c "import json; d=json.load(open('gpurun_out/r3k_bench_C3.json')); print(d['ms_per_step'], d['value'])"
