mkdir -p gpurun_out/r42
for v in a2 a2m4 a2m5 a3m4 cca a2 a2m4 a2m5 a3m4 cca; do EDL_LIB=variants/lib_$v.so timeout 300 python tools/ntt_bench.py >> gpurun_out/r42/nb.log 2>&1; done
