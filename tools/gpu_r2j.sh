#!/bin/bash
# final round-2 evidence: full GPU suite, smoke, default bench line (C5) + reference arm, C2 line
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/gpu_tests_r2j.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests_r2j.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2j.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_r2j.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_C5_r2j.json 2> gpurun_out/bench_C5_r2j.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref_C5_r2j.json 2> gpurun_out/ref_C5_r2j.err; echo "ref rc=$?"
timeout 300 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C2_r2j.json 2> gpurun_out/bench_C2_r2j.err; echo "C2 rc=$?"
python bench.py --gpus 2 > gpurun_out/bench_g2_r2j.json 2>&1; echo "gpus2 rc=$? (expected 1 on a 1-GPU box)"; tail -1 gpurun_out/bench_g2_r2j.json
