#!/bin/bash
# full GPU suite + default bench line on the slab route
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/gpu_tests_r2h.log 2>&1; echo "tests rc=$?"; grep -E "^FAILED|passed|failed" gpurun_out/gpu_tests_r2h.log | tail -8
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C5_r2h.json 2> gpurun_out/bench_C5_r2h.err; echo "bench rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_C5_r2h.json'))
print(d['ms_per_step'], d['value'], d['e2e']['ms_per_step']); print(json.dumps(d['roofline'])[:600]); print(json.dumps(d['rho_contraction'])[:900]); print(d['parity_prefix'])"
