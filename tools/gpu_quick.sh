# quick loop: slab-route parity (C3, C5 fixtures, small d=3 paths) + the fused-pass timing of C5 and C3
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fixtures.py tests/test_gpu_parity.py -q --timeout 600 > gpurun_out/gpu_quick.log 2>&1; echo "tests rc=$?"; tail -6 gpurun_out/gpu_quick.log
timeout 600 python tools/parity_report.py C3 C5 > gpurun_out/parity_quick.jsonl 2>&1; echo "parity rc=$?"
python - <<'PY'
import json
for l in open('gpurun_out/parity_quick.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l[:300]); continue
    print(d['config'], d['models'], 'coef %.2e obj %.2e dev %.2e'%(d['max_coef_rel'], d['max_obj_rel'], d['max_dev_rel']), d['all_supports_equal'], d['all_iteration_counts_equal'])
PY
(timeout 300 python tools/time_kernel.py --config C5; timeout 300 python tools/time_kernel.py --config C3) > gpurun_out/time_kernel.log 2>&1; echo "tk rc=$?"; tail -12 gpurun_out/time_kernel.log
