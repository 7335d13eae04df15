mkdir -p gpurun_out/r38
for v in default xs na default xs na; do if [ $v = default ]; then unset EDL_LIB; else export EDL_LIB=variants/lib_$v.so; fi
  timeout 300 python tools/path_rates.py >> gpurun_out/r38/path.log 2>&1
done
