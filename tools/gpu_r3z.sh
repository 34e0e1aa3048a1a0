#!/bin/bash
# final evidence of this pass: full GPU suite, smoke, default bench line (C5) + reference arm, C2-C4 lines, ncu --set full of the slab pass

mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/gpu_tests_r3z.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/gpu_tests_r3z.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r3z.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_r3z.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_C5_r3z.json 2> gpurun_out/bench_C5_r3z.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref_C5_r3z.json 2> gpurun_out/ref_C5_r3z.err; echo "ref rc=$?"
for c in C2 C3 C4; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${c}_r3z.json 2> gpurun_out/bench_${c}_r3z.err; echo "$c rc=$?"; done

timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_slab -s 2 -c 1 -o gpurun_out/r03_C5_k_slab4_last python tools/time_kernel.py --config C5 --which 0 --reps 3 > gpurun_out/ncu_slab_r3z.log 2>&1; echo "ncu slab rc=$?"
