#!/bin/bash
export KG_DEV=1
for pf in 0 4; do for d in 23 22 6 20 7; do
  echo "PF=$pf DBG=$d"; KG_SLAB_PF=$pf KG_SLAB_DBG=$d timeout 300 python tools/time_kernel.py --config C5 --which 0 --reps 20
done; done
