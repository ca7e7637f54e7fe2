out=gpurun_out; mkdir -p $out; rm -f $out/r2x.txt
timeout 1500 python -m pytest tests/test_gpu_dist.py tests/test_gpu_fullsize.py -x -q -k "peer or distributed" > $out/r2x_tests.log 2>&1; echo "rc=$?" >> $out/r2x_tests.log
echo "== exact" >> $out/r2x.txt; timeout 600 python scripts/scale_probe.py >> $out/r2x.txt 2>&1
tail -3 $out/r2x_tests.log; cat $out/r2x.txt
