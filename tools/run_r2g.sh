for v in main g0 g32 g128; do
  if [ $v = main ]; then L=paper_2110_13638_b200/libedl.so; else L=variants/$v.so; fi
  EDL_LIB=$L timeout 300 python tools/ntt_bench.py > gpurun_out/nb_$v.json 2> gpurun_out/nb_$v.err; echo "$v bench rc=$?" >> gpurun_out/summary.log
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_configs.py -q -x -k "layers or relin or c1_full or c3_full or activations or dense" > gpurun_out/pt.log 2>&1; echo "pytest rc=$?" >> gpurun_out/summary.log
