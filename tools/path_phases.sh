#!/bin/bash
# GPU-box recipe: k_gauss_path per-phase cycle counts (KG_DEV=1 KG_PATH_DBG=128) for
# the Gaussian whole-path configs; extra debug bits via DBG_EXTRA.
for bs in ${BS_LIST:-256 512}; do
  for c in ${CFGS:-C1 C2}; do
    echo "== bs=$bs $c"
    KG_DEV=1 KG_PATH_BS=$bs KG_PATH_DBG=$((128 + ${DBG_EXTRA:-0})) timeout 120 python tools/prof_path.py --config $c --paths 2 2>&1 | tail -3
  done
done
