for v in main split; do
  if [ $v = main ]; then L=paper_2110_13638_b200/libedl.so; else L=variants/$v.so; fi
  EDL_LIB=$L timeout 300 python tools/ntt_bench.py > gpurun_out/nb_$v.json 2> gpurun_out/nb_$v.err; echo "$v bench rc=$?" >> gpurun_out/summary.log
done
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/summary.log
