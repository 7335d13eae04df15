O=gpurun_out/${RUNDIR:-r75}; mkdir -p $O
for nf in 2 3 4; do for k in 10 20; do
timeout 900 python bench.py --no-c2 --no-c3 --no-cpu-baseline --no-e2e --inflight $nf --steps $k > $O/bench_i${nf}_k${k}.json 2> $O/bench_i${nf}_k${k}.err; echo "inflight=$nf steps=$k rc=$?" >> $O/summary.log
done; done
