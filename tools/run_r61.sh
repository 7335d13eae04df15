O=gpurun_out/${RUNDIR:-r61}; mkdir -p $O
for v in base default cbank cbank5; do
  if [ $v = default ]; then L=""; elif [ $v = base ]; then L=variants/lib_base.so; else L=variants/lib_$v.so; fi
  EDL_LIB=$L timeout 900 python -m pytest tests -q -m gpu -x -k "cc or c1_full or c3_full or dense or layers or extreme" > $O/pytest_$v.log 2>&1; echo "$v pytest rc=$?" >> $O/summary.log
  for rep in 1 2; do
  EDL_LIB=$L timeout 300 python tools/ntt_bench.py > $O/nb_$v.log 2>&1; python -c "
import json; d=json.loads(open('$O/nb_$v.log').read().strip().splitlines()[-1]); print('$v', round(d['c1_step_ms'],4), 'cc', d['c1_kernels_ms']['k_cc_mac'], 'dense', d['c1_kernels_ms']['k_dense_mac'])" >> $O/summary.log
  done
done
