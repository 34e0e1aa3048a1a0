#!/bin/bash
mkdir -p gpurun_out
export KG_DEV=1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "slab or poisson" --timeout 600 > gpurun_out/r3f_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r3f_tests.log
for pf in 0 4; do echo "K4 PF=$pf"; KG_SLAB_PF=$pf timeout 300 python tools/time_kernel.py --config C5 --which 0 --reps 20; done
for d in 2 4 16; do echo "PF=4 DBG=$d"; KG_SLAB_PF=4 KG_SLAB_DBG=$d timeout 300 python tools/time_kernel.py --config C5 --which 0 --reps 20; done
echo "C3 K4"; KG_SLAB_PF=4 timeout 300 python tools/time_kernel.py --config C3 --which 0 --reps 20
