#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/e2e_breakdown.py --config C4 --reps 4 2>&1 | head -5
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/r3r_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r3r_tests.log
for c in C4 C2; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r3r_bench_$c.json 2> gpurun_out/r3r.err; python tools/bench_brief.py gpurun_out/r3r_bench_$c.json; done
