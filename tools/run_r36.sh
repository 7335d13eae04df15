mkdir -p gpurun_out/r36
timeout 300 python tools/path_rates.py >> gpurun_out/r36/path.log 2>&1
timeout 300 python tools/ntt_bench.py >> gpurun_out/r36/nb.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_configs.py -q -x > gpurun_out/r36/pt.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r36/pt.log
timeout 300 python tools/ntt_bench.py >> gpurun_out/r36/nb.log 2>&1
timeout 300 python tools/path_rates.py >> gpurun_out/r36/path.log 2>&1
