#!/bin/bash
# k_slab2: mbarrier hand-over (default) vs named barriers (KG_SLAB_NB=1)
mkdir -p gpurun_out
export KG_DEV=1
for pf in 4 8; do for vs in 2 3; do
  echo "MB VS=$vs PF=$pf"; KG_SLAB_VS=$vs KG_SLAB_PF=$pf timeout 300 python tools/time_kernel.py --config C5 --which 0 --reps 20
done; done
echo "NB PF=4"; KG_SLAB_NB=1 KG_SLAB_PF=4 timeout 300 python tools/time_kernel.py --config C5 --which 0 --reps 20
echo "C3 MB"; KG_SLAB_PF=4 timeout 300 python tools/time_kernel.py --config C3 --which 0 --reps 20
echo "C3 NB"; KG_SLAB_NB=1 KG_SLAB_PF=4 timeout 300 python tools/time_kernel.py --config C3 --which 0 --reps 20
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "slab or poisson" --timeout 600 > gpurun_out/r3d_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r3d_tests.log
