#!/bin/bash
mkdir -p gpurun_out
for i in 1 2; do
KG_DEV=1 KG_NO_PDL=1 timeout 300 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r3l_C3_nopdl.json 2> gpurun_out/r3l.err; python tools/bench_brief.py gpurun_out/r3l_C3_nopdl.json
timeout 300 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r3l_C3.json 2> gpurun_out/r3l.err; python tools/bench_brief.py gpurun_out/r3l_C3.json
done
