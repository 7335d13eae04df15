mkdir -p gpurun_out/r34
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_configs.py -q -x -k "cc or layers or c1_full or extreme or sharded" > gpurun_out/r34/pt.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r34/pt.log
timeout 300 python tools/ntt_bench.py >> gpurun_out/r34/nb.log 2>&1
timeout 300 python tools/ntt_bench.py >> gpurun_out/r34/nb.log 2>&1
