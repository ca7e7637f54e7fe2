# round-2 check: exact reductions (tests + A/B vs the tree variant)
out=gpurun_out; mkdir -p $out
timeout 300 python scripts/ab_cg.py > $out/r2b_ab.txt 2>&1
LBK_LIB=$PWD/_variants/liblbk_LBK_RED_TREE.so timeout 300 python scripts/ab_cg.py >> $out/r2b_ab.txt 2>&1
timeout 300 python scripts/ab_cg.py >> $out/r2b_ab.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_exact.py -x -q > $out/r2b_exact.log 2>&1; echo "rc=$?" >> $out/r2b_exact.log
timeout 1500 python -m pytest tests -q -m gpu --deselect tests/test_gpu_exact.py > $out/r2b_pytest.log 2>&1; echo "rc=$?" >> $out/r2b_pytest.log
cat $out/r2b_ab.txt; tail -15 $out/r2b_exact.log; tail -25 $out/r2b_pytest.log
