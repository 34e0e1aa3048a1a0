#!/bin/bash
# GPU-box recipe: k_gauss_path variants (KG_DEV=1 KG_PATH_BS workers, KG_PATH_CW control
# warp) on the Gaussian whole-path configs, plus the Gaussian path parity tests.
mkdir -p gpurun_out
for cw in ${CW_LIST:-1 0}; do
for bs in ${BS_LIST:-256 512}; do
  for c in ${CFGS:-C1 C2 C4}; do
    echo "== cw=$cw bs=$bs $c"
    KG_DEV=1 KG_PATH_CW=$cw KG_PATH_BS=$bs KG_PATH_DBG=${DBG:-0} timeout 120 python tools/prof_path.py --config $c --paths 3 2>&1 | tail -${TAILN:-1}
  done
  KG_DEV=1 KG_PATH_CW=$cw KG_PATH_BS=$bs timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "gaussian or gram or c2 or deterministic" 2>&1 | tail -${TAILN:-1}
done
done
