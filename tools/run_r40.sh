mkdir -p gpurun_out/r40
for v in l8 default l8 default; do if [ $v = default ]; then unset EDL_LIB; else export EDL_LIB=variants/lib_$v.so; fi
  timeout 300 python tools/path_rates.py >> gpurun_out/r40/path.log 2>&1
  timeout 300 python tools/ntt_bench.py >> gpurun_out/r40/nb.log 2>&1
done
EDL_LIB=variants/lib_l8.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_configs.py -q -k "(ntt and 14) or relin or c1_full or extreme or rescale" > gpurun_out/r40/pt.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r40/pt.log
