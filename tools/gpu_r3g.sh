#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_slab -s 2 -c 1 -o gpurun_out/r03_C5_k_slab4c python tools/time_kernel.py --config C5 --which 0 --reps 3 > gpurun_out/ncu_slab_r3g2.log 2>&1; echo "ncu full rc=$?"
