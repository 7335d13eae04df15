timeout 300 python tools/ntt_bench.py > gpurun_out/nb.json 2> gpurun_out/nb.err; echo "bench rc=$?" >> gpurun_out/summary.log
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/summary.log
