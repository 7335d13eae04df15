O=gpurun_out/${RUNDIR:-r51}; mkdir -p $O
timeout 300 python tools/ntt_bench.py > $O/nb_base.log 2>&1; echo "nb base rc=$?" >> $O/summary.log
EDL_PDL=1 timeout 300 python tools/ntt_bench.py > $O/nb_pdl.log 2>&1; echo "nb pdl rc=$?" >> $O/summary.log
EDL_PDL=1 EDL_LIB=variants/lib_pdltrig.so timeout 300 python tools/ntt_bench.py > $O/nb_pdltrig.log 2>&1; echo "nb pdltrig rc=$?" >> $O/summary.log
EDL_PDL=1 timeout 2400 python -m pytest tests -q -m gpu -x > $O/pytest_gpu_pdl.log 2>&1; echo "pytest pdl rc=$?" >> $O/summary.log
EDL_PDL=1 EDL_LIB=variants/lib_pdltrig.so timeout 900 python -m pytest tests/test_gpu_full_configs.py -q -m gpu -x -k c1 > $O/pytest_trig.log 2>&1; echo "pytest trig rc=$?" >> $O/summary.log
timeout 300 python tools/ntt_bench.py > $O/nb_base2.log 2>&1; echo "nb base2 rc=$?" >> $O/summary.log
EDL_PDL=1 timeout 300 python tools/ntt_bench.py > $O/nb_pdl2.log 2>&1; echo "nb pdl2 rc=$?" >> $O/summary.log
EDL_PDL=1 EDL_LIB=variants/lib_pdltrig.so timeout 300 python tools/ntt_bench.py > $O/nb_pdltrig2.log 2>&1; echo "nb pdltrig2 rc=$?" >> $O/summary.log
