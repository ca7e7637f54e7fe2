out=gpurun_out; mkdir -p $out; rm -f $out/r2v.txt
timeout 900 python -m pytest tests/test_gpu_exact.py tests/test_gpu_dist.py -x -q > $out/r2v_tests.log 2>&1; echo "rc=$?" >> $out/r2v_tests.log
timeout 300 python scripts/ab_cg.py >> $out/r2v.txt 2>&1
LBK_LIB=$PWD/_variants/liblbk_LBK_RED_TREE.so timeout 300 python scripts/ab_cg.py >> $out/r2v.txt 2>&1
echo "== exact" >> $out/r2v.txt; timeout 600 python scripts/scale_probe.py >> $out/r2v.txt 2>&1
echo "== tree" >> $out/r2v.txt; LBK_LIB=$PWD/_variants/liblbk_LBK_RED_TREE.so timeout 600 python scripts/scale_probe.py >> $out/r2v.txt 2>&1
tail -3 $out/r2v_tests.log; cat $out/r2v.txt
