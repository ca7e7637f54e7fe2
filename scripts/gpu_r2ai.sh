out=gpurun_out; mkdir -p $out; rm -f $out/r2ai.txt
timeout 900 python -m pytest tests/test_gpu_exact.py tests/test_gpu_solver.py -x -q > $out/r2ai_pytest.log 2>&1; echo "pytest rc=$?" >> $out/r2ai.txt
tail -5 $out/r2ai_pytest.log >> $out/r2ai.txt
timeout 600 python -m pytest tests/test_gpu_fullsize.py -x -q -k "cfg4 or cfg5" >> $out/r2ai_pytest.log 2>&1; echo "fullsize rc=$?" >> $out/r2ai.txt
tail -3 $out/r2ai_pytest.log >> $out/r2ai.txt
timeout 300 python scripts/ab_cg.py >> $out/r2ai.txt 2>&1
LBK_CG2=0 timeout 300 python scripts/ab_cg.py >> $out/r2ai.txt 2>&1
timeout 300 python scripts/ab_cg.py >> $out/r2ai.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:'csr_stream|vec_kernel' --csv --log-file $out/r2ai_ncu.csv python scripts/prof_k1.py > /dev/null 2>&1
python scripts/ncu_table.py $out/r2ai_ncu.csv >> $out/r2ai.txt 2>&1
cat $out/r2ai.txt
