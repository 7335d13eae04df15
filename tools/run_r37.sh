mkdir -p gpurun_out/r37
timeout 300 python tools/path_rates.py >> gpurun_out/r37/path.log 2>&1
timeout 300 python tools/ntt_bench.py >> gpurun_out/r37/nb.log 2>&1
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/r37/pt.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r37/pt.log
timeout 300 python tools/ntt_bench.py >> gpurun_out/r37/nb.log 2>&1
