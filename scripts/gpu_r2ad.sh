out=gpurun_out; mkdir -p $out; rm -f $out/r2ad.txt
timeout 900 python -m pytest tests/test_gpu_exact.py -x -q > $out/r2ad_tests.log 2>&1; echo "rc=$?" >> $out/r2ad_tests.log
timeout 300 python scripts/ab_cg.py >> $out/r2ad.txt 2>&1
timeout 300 python scripts/ab_cg.py >> $out/r2ad.txt 2>&1
tail -2 $out/r2ad_tests.log; cat $out/r2ad.txt
