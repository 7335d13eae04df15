timeout 300 python tools/ntt_bench.py > gpurun_out/nb.json 2> gpurun_out/nb.err; echo "bench rc=$?" >> gpurun_out/summary.log
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_configs.py -q -x -k "relin or layers or c1_full or activations or rotate or keyswitch or chunked or raise" > gpurun_out/pt.log 2>&1; echo "pytest rc=$?" >> gpurun_out/summary.log
