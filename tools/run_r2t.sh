mkdir -p gpurun_out/r2t
python tools/ntt_path_run.py fp40 fwd > gpurun_out/r2t/plain.log 2>&1 || exit 1
export EDL_LIB=variants/lib_p4.so
for pd in "fp40 fwd" "fp40 inv" "int60 fwd"; do set -- $pd
  timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:k_ntt_limbs -s 1 -c 1 -o /tmp/n_$1_$2 python tools/ntt_path_run.py $1 $2 > gpurun_out/r2t/ncu_$1_$2.log 2>&1
  python tools/ncu_src.py /tmp/n_$1_$2.ncu-rep k_ntt_limbs 40 > gpurun_out/r2t/src_$1_$2.txt 2>&1
  ncu -i /tmp/n_$1_$2.ncu-rep --page details --csv > gpurun_out/r2t/det_$1_$2.csv 2>&1
done
