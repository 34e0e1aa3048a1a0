mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_sharded_product.py tests/test_gpu_parity.py -q --timeout 600 -k "sharded or shard or world" > gpurun_out/gpu_shard.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/gpu_shard.log
