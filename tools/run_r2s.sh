mkdir -p gpurun_out/r2s
for v in b14 p4 p5 b14 p5; do EDL_LIB=variants/lib_$v.so timeout 300 python tools/path_rates.py >> gpurun_out/r2s/path.log 2>&1; done
