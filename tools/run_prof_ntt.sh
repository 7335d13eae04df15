for v in base14 persist14; do
  EDL_LIB=variants/$v.so python tools/prof_ntt.py > gpurun_out/pn_$v.log 2>&1 && \
  EDL_LIB=variants/$v.so ncu --set full --clock-control none --import-source on -k regex:k_ntt_limbs -s 2 -c 2 -o gpurun_out/pn_$v python tools/prof_ntt.py > gpurun_out/pn_ncu_$v.log 2>&1
done
