mkdir -p gpurun_out/r2w
timeout 300 python tools/prof_step.py --step-only > gpurun_out/r2w/ps.log 2>&1 || exit 1
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:'k_(cc_mac|dense_mac|relin_mac)' -c 4 -o /tmp/mac python tools/prof_step.py --step-only > gpurun_out/r2w/ncu.log 2>&1
for k in k_cc_mac k_dense_mac k_relin_mac; do python tools/ncu_src.py /tmp/mac.ncu-rep $k 30 > gpurun_out/r2w/src_$k.txt 2>&1; done
python tools/ncu_step_summary.py /tmp/mac.ncu-rep gpurun_out/r2w > /dev/null 2>&1
cp /tmp/mac.ncu-rep gpurun_out/r2w/ 2>/dev/null
