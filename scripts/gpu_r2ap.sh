out=gpurun_out; mkdir -p $out; rm -f $out/r2ap.txt
timeout 900 python -m pytest tests/test_gpu_exact.py tests/test_gpu_solver.py tests/test_gpu_dist.py -x -q > $out/r2ap_pytest.log 2>&1; echo "pytest rc=$?" >> $out/r2ap.txt; tail -2 $out/r2ap_pytest.log >> $out/r2ap.txt
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "cfg4 or cfg5" >> $out/r2ap_pytest.log 2>&1; echo "fullsize rc=$?" >> $out/r2ap.txt; tail -2 $out/r2ap_pytest.log >> $out/r2ap.txt
for rep in 1 2; do
for lib in "" _variants/*.so; do
  if [ -n "$lib" ]; then export LBK_LIB=$PWD/$lib; else unset LBK_LIB; fi
  timeout 300 python scripts/ab_cg.py >> $out/r2ap.txt 2>&1
done
done
cat $out/r2ap.txt
