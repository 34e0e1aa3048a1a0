#!/bin/bash
# GPU-box recipe: default bench line, then the ncu launch list of the same command.
# usage: bash tools/gpu_bench.sh [config]
cfg=${1:-C2}
mkdir -p gpurun_out
python bench.py --config "$cfg" --steps 5 --warmup 3 > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err
rc=$?
echo "bench rc=$rc"
tail -c 4000 gpurun_out/bench_$cfg.json
tail -5 gpurun_out/bench_$cfg.err
if [ $rc -eq 0 ]; then
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$cfg.csv \
    python bench.py --config "$cfg" --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_$cfg.log 2>&1
  echo "ncu rc=$?"
fi
