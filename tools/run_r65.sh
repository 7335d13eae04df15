O=gpurun_out/${RUNDIR:-r65}; mkdir -p $O
for v in ${VARS:-base bulk bulk3}; do
  L=variants/lib_$v.so
  EDL_LIB=$L timeout 900 python -m pytest tests -q -m gpu -x -k "relin or c1_full or rotate or keyswitch or mixed or activations" > $O/pytest_$v.log 2>&1; echo "$v pytest rc=$?" >> $O/summary.log
  for rep in 1 2; do
  EDL_LIB=$L timeout 300 python tools/ntt_bench.py > $O/nb_$v.log 2>&1; python -c "
import json; d=json.loads(open('$O/nb_$v.log').read().strip().splitlines()[-1]); print('$v', round(d['c1_step_ms'],4), d['c1_kernels_ms'])" >> $O/summary.log
  done
done
