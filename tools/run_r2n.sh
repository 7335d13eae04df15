python tools/prof_step.py --step-only > gpurun_out/ps.log 2>&1 && \
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:'k_relin_(modup|moddown_ntt)' -c 2 -o /tmp/s2 python tools/prof_step.py --step-only > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/summary.log
for k in k_relin_modup k_relin_moddown_ntt k_rescale_ntt k_relin_intt_d2; do python tools/ncu_src.py /tmp/s2.ncu-rep $k 30 > gpurun_out/src_$k.txt 2>&1; done
python tools/ncu_step_summary.py /tmp/s2.ncu-rep gpurun_out/sum > /dev/null 2>&1
