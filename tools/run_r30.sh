mkdir -p gpurun_out/r30
for v in c6 c5 c6 c5; do EDL_LIB=variants/lib_$v.so timeout 300 python tools/ntt_bench.py >> gpurun_out/r30/nb.log 2>&1; done
