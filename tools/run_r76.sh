O=gpurun_out/${RUNDIR:-r76}; mkdir -p $O
timeout 900 python bench.py --no-c2 --no-c3 --no-cpu-baseline --no-e2e > $O/bench_k5.json 2> $O/bench_k5.err; echo "k5 rc=$?" >> $O/summary.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/summary.log
timeout 600 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-c2 --no-c3 > $O/b_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-c2 --no-c3 > $O/ncu_launch.log 2>&1; echo "launches rc=$?" >> $O/summary.log
