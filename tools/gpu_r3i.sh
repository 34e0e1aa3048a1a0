#!/bin/bash
# full GPU suite + smoke + bench lines with k_slab4
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 > gpurun_out/r3i_gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r3i_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3i_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r3i_smoke.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r3i_bench_C5.json 2> gpurun_out/r3i_bench_C5.err; echo "bench rc=$?"; cat gpurun_out/r3i_bench_C5.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['e2e'], d['roofline']['avg_launch_ms'], d['roofline']['frac'], d.get('parity_prefix'))"
timeout 300 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r3i_bench_C3.json 2> gpurun_out/r3i_bench_C3.err; echo "C3 rc=$?"; python -c "import json; d=json.load(open('gpurun_out/r3i_bench_C3.json')); print(d['ms_per_step'], d['value'])"
