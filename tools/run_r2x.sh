mkdir -p gpurun_out/r2x
for v in nc default nc default; do if [ $v = default ]; then unset EDL_LIB; else export EDL_LIB=variants/lib_$v.so; fi
  timeout 300 python tools/path_rates.py >> gpurun_out/r2x/path.log 2>&1
  timeout 300 python tools/ntt_bench.py >> gpurun_out/r2x/nb.log 2>&1
done
