mkdir -p gpurun_out/r32
export EDL_LIB=variants/lib_c6.so
timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:'k_(cc_mac|dense_mac)' -c 2 -o /tmp/cc6 python tools/prof_step.py --step-only > gpurun_out/r32/ncu.log 2>&1
python tools/ncu_src.py /tmp/cc6.ncu-rep k_cc_mac 30 > gpurun_out/r32/src_cc.txt 2>&1
python tools/ncu_src.py /tmp/cc6.ncu-rep k_dense_mac 30 > gpurun_out/r32/src_dense.txt 2>&1
python tools/ncu_step_summary.py /tmp/cc6.ncu-rep gpurun_out/r32 > /dev/null 2>&1
