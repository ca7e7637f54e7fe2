out=gpurun_out; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_dist.py tests/test_gpu_exact.py -x -q > $out/r2ae.log 2>&1; echo "rc=$?" >> $out/r2ae.log
tail -3 $out/r2ae.log
