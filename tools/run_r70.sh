O=gpurun_out/${RUNDIR:-r70}; mkdir -p $O
timeout 900 python -m pytest tests -q -m gpu -x -k "two_contexts or c3_full" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/summary.log
timeout 900 python bench.py --no-c2 --no-c3 --no-cpu-baseline > $O/bench_i2.json 2> $O/bench_i2.err; echo "bench i2 rc=$?" >> $O/summary.log
timeout 900 python bench.py --no-c2 --no-c3 --no-cpu-baseline --inflight 1 > $O/bench_i1.json 2> $O/bench_i1.err; echo "bench i1 rc=$?" >> $O/summary.log
timeout 900 python bench.py --no-c2 --no-c3 --no-cpu-baseline --inflight 3 --steps 12 > $O/bench_i3.json 2> $O/bench_i3.err; echo "bench i3 rc=$?" >> $O/summary.log
