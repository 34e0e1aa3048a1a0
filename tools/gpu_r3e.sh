#!/bin/bash
# k_slab4 timing experiments (KG_SLAB_DBG bits: 1 no v loads, 2 tensor warps skip gather/Z, 4 row warps skip their FP64 work and stores, 16 tensor warps skip the U math)
export KG_DEV=1 KG_SLAB_PF=4
for d in 0 1 2 16 4 18 5 23; do
  echo "DBG=$d"; KG_SLAB_DBG=$d timeout 300 python tools/time_kernel.py --config C5 --which 0 --reps 20
done
