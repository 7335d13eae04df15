for v in "$@"; do EDL_LIB=variants/lib_$v.so timeout 300 python tools/ntt_bench.py > gpurun_out/nb_$v.log 2>&1; python -c "
import json,sys; d=json.loads(open('gpurun_out/nb_$v.log').read().strip().splitlines()[-1]); print('$v', {k:(round(v,3) if isinstance(v,float) else v) for k,v in d.items() if k!='lib'})" || tail -3 gpurun_out/nb_$v.log; done
