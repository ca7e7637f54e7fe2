out=gpurun_out; mkdir -p $out; rm -f $out/r2am.txt
timeout 900 python -m pytest tests/test_gpu_spmv.py -x -q > $out/r2am_pytest.log 2>&1; echo "pytest rc=$?" >> $out/r2am.txt; tail -2 $out/r2am_pytest.log >> $out/r2am.txt
for rep in 1; do
for lib in "" _variants/*.so; do
  if [ -n "$lib" ]; then export LBK_LIB=$PWD/$lib; else unset LBK_LIB; fi
  echo "lib=${lib:-default}" >> $out/r2am.txt
  timeout 300 python scripts/prof_pl.py >> $out/r2am.txt 2>&1
done
done
unset LBK_LIB
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k cfg3 >> $out/r2am_pytest.log 2>&1; echo "cfg3 full rc=$?" >> $out/r2am.txt; tail -2 $out/r2am_pytest.log >> $out/r2am.txt
cat $out/r2am.txt
