out=gpurun_out; mkdir -p $out; rm -f $out/r2al.txt
timeout 900 python -m pytest tests/test_gpu_spmv.py -x -q > $out/r2al_pytest.log 2>&1; echo "pytest rc=$?" >> $out/r2al.txt; tail -2 $out/r2al_pytest.log >> $out/r2al.txt
for rep in 1; do
for lib in "" _variants/*.so; do
  if [ -n "$lib" ]; then export LBK_LIB=$PWD/$lib; else unset LBK_LIB; fi
  echo "lib=${lib:-default}" >> $out/r2al.txt
  timeout 300 python scripts/prof_pl.py >> $out/r2al.txt 2>&1
done
done
unset LBK_LIB
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k cfg3 >> $out/r2al_pytest.log 2>&1; echo "cfg3 full rc=$?" >> $out/r2al.txt; tail -2 $out/r2al_pytest.log >> $out/r2al.txt
cat $out/r2al.txt
