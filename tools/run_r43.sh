O=gpurun_out/r43; mkdir -p $O
for v in dna default dna default; do if [ $v = default ]; then unset EDL_LIB; else export EDL_LIB=variants/lib_$v.so; fi
  timeout 300 python tools/ntt_bench.py >> $O/nb.log 2>&1
done
unset EDL_LIB
timeout 2400 python -m pytest tests -q -m gpu > $O/pt.log 2>&1; echo "pytest rc=$?" >> $O/pt.log
EDL_BENCH_EMULATE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 1 --no-e2e --no-c2 --no-c3 > $O/emul2.log 2>&1; echo "emul rc=$?" >> $O/pt.log
