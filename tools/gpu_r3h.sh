#!/bin/bash
export KG_DEV=1 KG_SLAB_PF=8
for d in 0 1 2 16 18 4 5 23; do
echo "DBG=$d"
KG_SLAB_DBG=$d timeout 300 python tools/time_kernel.py --config C5 --which 0 --reps 1 2>&1 | grep -v "^\[" | grep "warp 8:\|warp 9:\|warp 0:\|warp 1:\|which" | sort | uniq | head -12
done
