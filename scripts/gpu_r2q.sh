out=gpurun_out; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_mm_sweep.py tests/test_gpu_solver.py tests/test_gpu_spmv.py -q > $out/r2q_tests.log 2>&1; echo "rc=$?" >> $out/r2q_tests.log
timeout 900 python scripts/mm_sweep.py --generate /tmp/mmc --out $out/r2_mm_sweep > $out/r2q_sweep.txt 2>&1
tail -5 $out/r2q_tests.log; cat $out/r2q_sweep.txt
