mkdir -p gpurun_out/r41
for v in a3 a2 a4 default a3 a2 a4 default; do if [ $v = default ]; then unset EDL_LIB; else export EDL_LIB=variants/lib_$v.so; fi
  timeout 300 python tools/ntt_bench.py >> gpurun_out/r41/nb.log 2>&1
done
EDL_LIB=variants/lib_a3.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_configs.py -q -k "(relin and not large_n and not c2_chain and not mixed) or c1_full or extreme or keyswitch or rotate" > gpurun_out/r41/pt.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r41/pt.log
