mkdir -p gpurun_out/r2p
for v in base mix base mix; do EDL_LIB=variants/lib_$v.so timeout 300 python tools/ntt_bench.py > gpurun_out/r2p/nb_$v.log 2>&1; tail -1 gpurun_out/r2p/nb_$v.log >> gpurun_out/r2p/all.log; done
EDL_LIB=variants/lib_mix.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_configs.py -q -x -k "relin or c1_full or rescale" > gpurun_out/r2p/pt_mix.log 2>&1; echo "pytest mix rc=$?" >> gpurun_out/r2p/all.log
