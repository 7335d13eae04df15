mkdir -p gpurun_out/r2
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2/bench.json 2> gpurun_out/r2/bench.err; echo "bench rc=$?" >> gpurun_out/summary.log
timeout 300 python tools/prof_step.py --step-only > gpurun_out/r2/ps.log 2>&1 && \
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:'k_(cc|rescale|relin|dense|add)' -o /tmp/step python tools/prof_step.py --step-only > gpurun_out/r2/ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/summary.log
python tools/ncu_step_summary.py /tmp/step.ncu-rep gpurun_out/r2 > /dev/null 2>&1
for k in k_relin_modup k_rescale_ntt k_relin_moddown_ntt k_relin_mac k_cc_mac; do python tools/ncu_src.py /tmp/step.ncu-rep $k 25 > gpurun_out/r2/src_$k.txt 2>&1; done
timeout 600 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-c2 --no-c3 > gpurun_out/r2/b_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-c2 --no-c3 > gpurun_out/r2/ncu_launch.log 2>&1; echo "launches rc=$?" >> gpurun_out/summary.log
