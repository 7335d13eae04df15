mkdir -p gpurun_out/r2q
for i in 1 2; do EDL_BENCH_ENVS="EDL_RAISE_FUSED=1" timeout 300 python tools/ntt_bench.py > gpurun_out/r2q/nb_raise$i.log 2>&1; tail -1 gpurun_out/r2q/nb_raise$i.log >> gpurun_out/r2q/all.log; done
