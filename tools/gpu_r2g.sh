#!/bin/bash
# round-2 evidence pass: full GPU suite, default bench (C5) + reference arm, launch list of the bench command
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/gpu_tests_r2g.log 2>&1; echo "tests rc=$?"; tail -6 gpurun_out/gpu_tests_r2g.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_C5_r2g.json 2> gpurun_out/bench_C5_r2g.err; echo "bench rc=$?"; tail -c 3500 gpurun_out/bench_C5_r2g.json; tail -3 gpurun_out/bench_C5_r2g.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref_C5_r2g.json 2> gpurun_out/ref_C5_r2g.err; echo "ref rc=$?"; cat gpurun_out/ref_C5_r2g.json
KG_HOST_LOOP=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C5_r2g.csv python tools/prof_path.py --config C5 --paths 1 --n-lambda 3 > gpurun_out/ncu_C5_r2g.log 2>&1; echo "ncu rc=$?"
python tools/launch_summary.py gpurun_out/launches_C5_r2g.csv | head -40
