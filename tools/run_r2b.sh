for v in ks8 noks14; do
  EDL_LIB=variants/$v.so timeout 300 python tools/ntt_bench.py > gpurun_out/nb_$v.json 2> gpurun_out/nb_$v.err; echo "$v bench rc=$?" >> gpurun_out/summary.log
done
EDL_LIB=variants/ks8.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "mul_relin_bit_exact or mul_relin_c2 or two_stream or mixed_levels" > gpurun_out/pt_ks8.log 2>&1; echo "ks8 pytest rc=$?" >> gpurun_out/summary.log
EDL_LIB=variants/ks8.so python tools/prof_step.py > gpurun_out/ps.log 2>&1 && EDL_LIB=variants/ks8.so ncu --set full --clock-control none --import-source on -k regex:"k_relin_ks" -c 2 -o /tmp/ks8 python tools/prof_step.py > gpurun_out/ncu_ks8.log 2>&1
python tools/ncu_src.py /tmp/ks8.ncu-rep k_relin_ks 40 > gpurun_out/src_ks8.txt 2>&1
ncu -i /tmp/ks8.ncu-rep --page raw --csv > gpurun_out/raw_ks8.csv 2>&1
