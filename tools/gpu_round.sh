#!/bin/bash
# GPU-box recipe for a round's evidence: full GPU test suite, the default bench
# line (C2) and the other configs, the ncu launch list of the default bench
# command, and one --set full capture of the C2 whole-path kernel.
mkdir -p gpurun_out
timeout 700 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/gpu_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests.log
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err
echo "bench rc=$?"
for c in C1 C3 C4 C5; do
  timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "$c rc=$?"
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C2.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo "ncu launches rc=$?"
timeout 400 ncu --set full --import-source on --clock-control none -k regex:k_gauss_path -c 1 \
  -o gpurun_out/r01_c2_path_final python tools/prof_path.py --config C2 --paths 1 > gpurun_out/ncu_path.log 2>&1
echo "ncu path rc=$?"
KG_HOST_LOOP=1 timeout 400 ncu --set full --clock-control none -k regex:k_contract_gb -s 4 -c 2 \
  -o gpurun_out/r01_c5_contract_gb python tools/prof_path.py --config C5 --paths 1 --n-lambda 2 > gpurun_out/ncu_gb.log 2>&1
echo "ncu contract_gb rc=$?"
