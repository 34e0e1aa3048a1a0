nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1700 python -m pytest tests -m gpu -q --timeout 900 -k "not C5" > gpurun_out/gpu_tests_r2a.log 2>&1
echo "tests rc=$?"; tail -15 gpurun_out/gpu_tests_r2a.log
timeout 900 python tools/parity_report.py C1 C2 C3 C4 > gpurun_out/parity_r2a.jsonl 2>&1; echo "parity rc=$?"
