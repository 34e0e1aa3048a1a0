#!/bin/bash
# final round-2 evidence: full GPU suite, smoke, default bench line (C5) + reference arm, C2 line,
# C5 launch list with DRAM bytes, ncu --set full of k_slab
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/gpu_tests_r2k.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/gpu_tests_r2k.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2k.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_r2k.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_C5_r2k.json 2> gpurun_out/bench_C5_r2k.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref_C5_r2k.json 2> gpurun_out/ref_C5_r2k.err; echo "ref rc=$?"
for c in C2 C3 C4; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${c}_r2k.json 2> gpurun_out/bench_${c}_r2k.err; echo "$c rc=$?"; done
KG_HOST_LOOP=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_C5_r2k.csv python tools/prof_path.py --config C5 --paths 1 --n-lambda 3 > gpurun_out/ncu_C5_r2k.log 2>&1; echo "ncu list rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_slab -s 2 -c 1 -o gpurun_out/r02_C5_k_slab_final python tools/time_kernel.py --config C5 --which 0 --reps 3 > gpurun_out/ncu_slab_r2k.log 2>&1; echo "ncu slab rc=$?"
