O=gpurun_out/${RUNDIR:-r66}; mkdir -p $O
timeout 1200 python -m pytest tests -q -m gpu -x -k "dense or c3_full or c1_full or layers or extreme or c0 or c4" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/summary.log
for L in variants/lib_base.so ""; do
EDL_LIB=$L timeout 600 python tools/c3_bench.py > $O/c3_$(basename "${L:-default}" .so).json 2>&1; echo "c3 $L rc=$?" >> $O/summary.log
done
