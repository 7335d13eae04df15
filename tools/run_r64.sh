O=gpurun_out/${RUNDIR:-r64}; mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/summary.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/ref.json 2> $O/ref.err; echo "ref rc=$?" >> $O/summary.log
EDL_BENCH_EMULATE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 > $O/emul2.json 2> $O/emul2.err; echo "emul2 rc=$?" >> $O/summary.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench default rc=$?" >> $O/summary.log
