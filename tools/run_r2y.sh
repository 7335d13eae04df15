mkdir -p gpurun_out/r2y
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_configs.py -q -x -k "cc or layers or c1_full or extreme or sharded or c3" > gpurun_out/r2y/pt.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2y/pt.log
timeout 300 python tools/ntt_bench.py >> gpurun_out/r2y/nb.log 2>&1
timeout 300 python tools/ntt_bench.py >> gpurun_out/r2y/nb.log 2>&1
