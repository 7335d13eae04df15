mkdir -p gpurun_out/r31
for v in pf4 pfw7 c6 pf4 pfw7 c6; do EDL_LIB=variants/lib_$v.so timeout 300 python tools/ntt_bench.py >> gpurun_out/r31/nb.log 2>&1; done
