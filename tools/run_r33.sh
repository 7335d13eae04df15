mkdir -p gpurun_out/r33
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/r33/pt.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r33/pt.log
timeout 300 python tools/ntt_bench.py >> gpurun_out/r33/nb.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r33/bench.json 2> gpurun_out/r33/bench.err; echo "bench rc=$?" >> gpurun_out/r33/pt.log
