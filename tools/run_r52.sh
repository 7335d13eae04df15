O=gpurun_out/${RUNDIR:-r52}; mkdir -p $O
EDL_BENCH_ENVS="EDL_KS_FUSED=1;EDL_RAISE_FUSED=1" timeout 400 python tools/ntt_bench.py > $O/nb_default.log 2>&1; echo "nb rc=$?" >> $O/summary.log
EDL_PDL=0 timeout 300 python tools/ntt_bench.py > $O/nb_nopdl.log 2>&1; echo "nb nopdl rc=$?" >> $O/summary.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/summary.log
