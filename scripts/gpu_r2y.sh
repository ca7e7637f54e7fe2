out=gpurun_out; mkdir -p $out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:coo_stream -s 2 -c 1 -o $out/r2y_coo python scripts/prof_coo.py > /dev/null 2>&1
ncu -i $out/r2y_coo.ncu-rep --page details > $out/r2y_coo_details.txt 2>&1
ncu -i $out/r2y_coo.ncu-rep --page source --csv > $out/r2y_coo_source.csv 2>&1
rm -f $out/*.ncu-rep
