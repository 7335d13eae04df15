O=gpurun_out/r44; mkdir -p $O
for v in cts16 cts4 dna cts16 cts4 dna; do EDL_LIB=variants/lib_$v.so timeout 300 python tools/ntt_bench.py >> $O/nb.log 2>&1; done
