out=gpurun_out; mkdir -p $out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:csr_stream -s 3 -c 1 -o $out/r2o_pl python scripts/prof_pl.py csr > /dev/null 2>&1
ncu -i $out/r2o_pl.ncu-rep --page details > $out/r2o_pl_details.txt 2>&1
ncu -i $out/r2o_pl.ncu-rep --page source --csv > $out/r2o_pl_source.csv 2>&1
ncu -i $out/r2o_pl.ncu-rep --page raw --csv > $out/r2o_pl_raw.csv 2>&1
rm -f $out/*.ncu-rep
