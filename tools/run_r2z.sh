mkdir -p gpurun_out/r2z
timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:'k_cc_mac' -c 1 -o /tmp/cc4 python tools/prof_step.py --step-only > gpurun_out/r2z/ncu.log 2>&1
python tools/ncu_src.py /tmp/cc4.ncu-rep k_cc_mac 40 > gpurun_out/r2z/src_cc4.txt 2>&1
python tools/ncu_step_summary.py /tmp/cc4.ncu-rep gpurun_out/r2z > /dev/null 2>&1
for v in m1 m2 m1 m2; do EDL_LIB=variants/lib_$v.so timeout 300 python tools/ntt_bench.py >> gpurun_out/r2z/nb.log 2>&1; done
