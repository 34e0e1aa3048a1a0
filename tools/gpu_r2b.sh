# round-2 check: FP64 pipe peaks, fixture parity tests, the default bench line (C5) and the reference arm
mkdir -p gpurun_out profiles
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak tools/probes/fp64_peak.cu && /tmp/fp64_peak > gpurun_out/fp64_peaks.json; echo "fp64 rc=$?"; cat gpurun_out/fp64_peaks.json
timeout 900 python -m pytest tests/test_gpu_fixtures.py tests/test_armijo.py -q --timeout 600 > gpurun_out/gpu_fix_r2b.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/gpu_fix_r2b.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_C5_r2b.json 2> gpurun_out/bench_C5_r2b.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench_C5_r2b.json; tail -5 gpurun_out/bench_C5_r2b.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 2 > gpurun_out/ref_C5_r2b.json 2> gpurun_out/ref_C5_r2b.err; echo "ref rc=$?"; cat gpurun_out/ref_C5_r2b.json; tail -3 gpurun_out/ref_C5_r2b.err
python bench.py --gpus 2 > gpurun_out/bench_g2.json 2>&1; echo "gpus2 rc=$?"; tail -3 gpurun_out/bench_g2.json
