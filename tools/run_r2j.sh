for v in main shoup4; do
  if [ $v = main ]; then L=paper_2110_13638_b200/libedl.so; else L=variants/$v.so; fi
  EDL_LIB=$L timeout 300 python tools/ntt_bench.py > gpurun_out/nb_$v.json 2> gpurun_out/nb_$v.err; echo "$v bench rc=$?" >> gpurun_out/summary.log
  EDL_LIB=$L python -c "
import sys; sys.path.insert(0,'.')
from paper_2110_13638_b200 import edl
c=edl.Context(edl.params_from_depth(4)); print('$v', 'bfly q0', c.bfly_peak(0)/1e9, 'q1', c.bfly_peak(1)/1e9)" >> gpurun_out/summary.log 2>&1
done
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/summary.log
