out=gpurun_out; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/r2a_smi.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > $out/r2a_pytest.log 2>&1; echo "rc=$?" >> $out/r2a_pytest.log
timeout 600 python bench.py > $out/r2a_bench.json 2> $out/r2a_bench.err
timeout 300 python scripts/prof_pl.py > $out/r2a_pl.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:csr_stream -s 3 -c 1 -o $out/r2a_plcsr python scripts/prof_pl.py csr > /dev/null 2>&1
ncu -i $out/r2a_plcsr.ncu-rep --page raw --csv > $out/r2a_plcsr_raw.csv 2>&1
ncu -i $out/r2a_plcsr.ncu-rep --page details > $out/r2a_plcsr_details.txt 2>&1
rm -f $out/*.ncu-rep
tail -3 $out/r2a_pytest.log; cat $out/r2a_pl.txt; tail -c 3000 $out/r2a_bench.json
