O=gpurun_out/${RUNDIR:-r79}; mkdir -p $O
for v in base wpb7; do
  L=variants/lib_$v.so
  EDL_LIB=$L timeout 600 python -m pytest tests -q -m gpu -x -k "cc or c1_full" > $O/pytest_$v.log 2>&1; echo "$v pytest rc=$?" >> $O/summary.log
  for rep in 1 2; do
  EDL_LIB=$L timeout 300 python tools/ntt_bench.py > $O/nb_$v.log 2>&1; python -c "
import json; d=json.loads(open('$O/nb_$v.log').read().strip().splitlines()[-1]); print('$v', round(d['c1_step_ms'],4), 'cc', d['c1_kernels_ms']['k_cc_mac'])" >> $O/summary.log
  done
done
