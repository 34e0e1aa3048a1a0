#!/bin/bash
# k_slab2: v register stages (KG_SLAB_VS) x L2 prefetch distance (KG_SLAB_PF)
mkdir -p gpurun_out
export KG_DEV=1
for vs in 2 3; do for pf in 0 4 8 16 32; do
  echo "VS=$vs PF=$pf"; KG_SLAB_VS=$vs KG_SLAB_PF=$pf timeout 300 python tools/time_kernel.py --config C5 --which 0 --reps 20
done; done
KG_SLAB_VS=3 KG_SLAB_PF=8 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "slab or poisson" --timeout 600 > gpurun_out/r3c_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r3c_tests.log
