O=gpurun_out/${RUNDIR:-r60}; mkdir -p $O
timeout 2400 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/summary.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/summary.log
timeout 600 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-c2 --no-c3 > $O/b_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-c2 --no-c3 > $O/ncu_launch.log 2>&1; echo "launches rc=$?" >> $O/summary.log
timeout 300 python tools/prof_step.py --step-only > $O/ps.log 2>&1 && \
timeout 1500 ncu -f --set full --clock-control none --import-source on -k regex:'k_(cc|rescale|relin|dense|add)' -o /tmp/step python tools/prof_step.py --step-only > $O/ncu.log 2>&1; echo "ncu rc=$?" >> $O/summary.log
python tools/ncu_step_summary.py /tmp/step.ncu-rep $O > /dev/null 2>&1
for k in k_relin_modup k_rescale_ntt k_relin_moddown_ntt k_relin_mac k_cc_mac k_relin_intt_d2 k_relin_moddown_intt k_dense_mac k_rescale_intt; do python tools/ncu_src.py /tmp/step.ncu-rep $k 25 > $O/src_$k.txt 2>&1; done
