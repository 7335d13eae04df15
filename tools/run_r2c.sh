for v in ks8c noksc; do
  EDL_LIB=variants/$v.so timeout 300 python tools/ntt_bench.py > gpurun_out/nb_$v.json 2> gpurun_out/nb_$v.err; echo "$v bench rc=$?" >> gpurun_out/summary.log
  EDL_LIB=variants/$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "ntt_bit_exact and 14 or ntt_prime_classes and 14 or large_batch or mul_relin_bit_exact or two_stream or mixed_levels or layers_small or rotate_bit" > gpurun_out/pt_$v.log 2>&1; echo "$v pytest rc=$?" >> gpurun_out/summary.log
done
