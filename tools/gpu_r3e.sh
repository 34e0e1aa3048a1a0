#!/bin/bash
# k_slab2 timing experiments: which stage bounds the chunk (KG_SLAB_DBG bits: 1 no v loads, 2 tensor warps skip gather/Z, 4 no scatter FMAs, 8 no eta chain)
export KG_DEV=1 KG_SLAB_PF=4
for d in 0 1 2 4 8 3 5 12 13 15; do
  echo "DBG=$d"; KG_SLAB_DBG=$d timeout 300 python tools/time_kernel.py --config C5 --which 0 --reps 20
done
