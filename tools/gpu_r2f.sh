mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/gpu_tests_r2f.log 2>&1; echo "tests rc=$?"; tail -6 gpurun_out/gpu_tests_r2f.log
python tools/prof_path.py --config C5 --paths 2 2>&1 | tail -1
python tools/prof_path.py --config C3 --paths 3 2>&1 | tail -1
