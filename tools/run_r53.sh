O=gpurun_out/${RUNDIR:-r53}; mkdir -p $O
timeout 900 python -m pytest tests -q -m gpu -x -k "cc or c1 or cross" > $O/pytest_cc.log 2>&1; echo "pytest cc rc=$?" >> $O/summary.log
for v in default k0 default k0; do
  if [ $v = default ]; then L=""; else L=variants/lib_cc4k0.so; fi
  EDL_LIB=$L timeout 300 python tools/ntt_bench.py > $O/nb_$v.log 2>&1; python -c "
import json; d=json.loads(open('$O/nb_$v.log').read().strip().splitlines()[-1]); print('$v', round(d['c1_step_ms'],4), d['c1_kernels_ms']['k_cc_mac'])" >> $O/summary.log
done
