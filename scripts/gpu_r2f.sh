out=gpurun_out; mkdir -p $out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:vec_kernel -s 0 -c 1 -o $out/r2f_vec python scripts/prof_k1.py > /dev/null 2>&1
ncu -i $out/r2f_vec.ncu-rep --page details > $out/r2f_vec_details.txt 2>&1
ncu -i $out/r2f_vec.ncu-rep --page source --csv > $out/r2f_vec_source.csv 2>&1
ncu -i $out/r2f_vec.ncu-rep --page raw --csv > $out/r2f_vec_raw.csv 2>&1
rm -f $out/*.ncu-rep
