out=gpurun_out; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_exact.py -x -q > $out/r2l_exact.log 2>&1; echo "rc=$?" >> $out/r2l_exact.log
timeout 1800 python -m pytest tests -q -m gpu --deselect tests/test_gpu_exact.py > $out/r2l_pytest.log 2>&1; echo "rc=$?" >> $out/r2l_pytest.log
tail -5 $out/r2l_exact.log; tail -8 $out/r2l_pytest.log
