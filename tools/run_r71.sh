O=gpurun_out/${RUNDIR:-r71}; mkdir -p $O
for sp in 1 0; do for nf in 2 3; do
EDL_KS_SPLIT=$sp timeout 900 python bench.py --no-c2 --no-c3 --no-cpu-baseline --no-e2e --inflight $nf --steps 20 > $O/bench_s${sp}_i${nf}.json 2> $O/bench_s${sp}_i${nf}.err; echo "bench split=$sp inflight=$nf rc=$?" >> $O/summary.log
done; done
