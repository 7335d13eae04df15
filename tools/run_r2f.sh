EDL_BENCH_CHUNKS=24,32,48,64 timeout 600 python tools/ntt_bench.py > gpurun_out/nb_main.json 2> gpurun_out/nb_main.err; echo "bench rc=$?" >> gpurun_out/summary.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "chunked or fused_keyswitch or dense or layers or c0_end" > gpurun_out/pt.log 2>&1; echo "pytest rc=$?" >> gpurun_out/summary.log
