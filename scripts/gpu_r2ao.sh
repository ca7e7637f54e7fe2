out=gpurun_out; mkdir -p $out; rm -f $out/r2ao.txt
LBK_LIB=$PWD/_variants/liblbk_LBK_CG_SPLIT_P.so timeout 900 python -m pytest tests/test_gpu_exact.py -x -q -k "solver" > $out/r2ao_pytest.log 2>&1; echo "pytest(split) rc=$?" >> $out/r2ao.txt; tail -2 $out/r2ao_pytest.log >> $out/r2ao.txt
for rep in 1 2; do
for lib in "" _variants/*.so; do
  if [ -n "$lib" ]; then export LBK_LIB=$PWD/$lib; else unset LBK_LIB; fi
  timeout 300 python scripts/ab_cg.py >> $out/r2ao.txt 2>&1
done
done
cat $out/r2ao.txt
