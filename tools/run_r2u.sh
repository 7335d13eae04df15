mkdir -p gpurun_out/r2u
for v in nopf default pfp4 nopf default; do if [ $v = default ]; then unset EDL_LIB; else export EDL_LIB=variants/lib_$v.so; fi
  timeout 300 python tools/path_rates.py >> gpurun_out/r2u/path.log 2>&1
  timeout 300 python tools/ntt_bench.py >> gpurun_out/r2u/nb.log 2>&1
done
unset EDL_LIB
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_configs.py -q -x > gpurun_out/r2u/pt.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2u/pt.log
