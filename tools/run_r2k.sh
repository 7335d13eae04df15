EDL_LIB=variants/raise.so EDL_BENCH_ENVS="EDL_RAISE_FUSED=1" timeout 600 python tools/ntt_bench.py > gpurun_out/nb.json 2> gpurun_out/nb.err; echo "bench rc=$?" >> gpurun_out/summary.log
EDL_LIB=variants/raise.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fused_raise or fused_keyswitch" > gpurun_out/pt.log 2>&1; echo "pytest rc=$?" >> gpurun_out/summary.log
