mkdir -p gpurun_out/r2o
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/r2o/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2o/summary.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2o/bench.json 2> gpurun_out/r2o/bench.err; echo "bench rc=$?" >> gpurun_out/r2o/summary.log
timeout 600 python tools/ntt_bench.py > gpurun_out/r2o/ntt_bench.log 2>&1; echo "ntt rc=$?" >> gpurun_out/r2o/summary.log
