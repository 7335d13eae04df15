O=gpurun_out/${RUNDIR:-r50}; mkdir -p $O
timeout 2400 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/summary.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/summary.log
timeout 300 python tools/ntt_bench.py > $O/nb.log 2>&1; echo "nb rc=$?" >> $O/summary.log
