out=gpurun_out; mkdir -p $out; rm -f $out/r2aj.txt
timeout 900 python -m pytest tests/test_gpu_exact.py -x -q -k "solver or dist_bits" > $out/r2aj_pytest.log 2>&1; echo "pytest rc=$?" >> $out/r2aj.txt
tail -2 $out/r2aj_pytest.log >> $out/r2aj.txt
for lib in "" _variants/*.so; do
  if [ -n "$lib" ]; then export LBK_LIB=$PWD/$lib; else unset LBK_LIB; fi
  timeout 300 python scripts/ab_cg.py >> $out/r2aj.txt 2>&1
  timeout 300 python scripts/ab_spmv.py >> $out/r2aj.txt 2>&1
done
unset LBK_LIB
cat $out/r2aj.txt
