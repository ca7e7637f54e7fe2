out=gpurun_out; mkdir -p $out
timeout 300 python scripts/ab_cg.py > $out/r2c_ab.txt 2>&1
LBK_LIB=$PWD/_variants/liblbk_LBK_RED_TREE.so timeout 300 python scripts/ab_cg.py >> $out/r2c_ab.txt 2>&1
LBK_LIB=$PWD/_variants/liblbk_LBK_XRED_STATS.so timeout 300 python scripts/xred_stats.py >> $out/r2c_ab.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:csr_stream -s 9 -c 3 -o $out/r2c_cg python scripts/prof_k1.py > /dev/null 2>&1
ncu -i $out/r2c_cg.ncu-rep --page details > $out/r2c_cg_details.txt 2>&1
ncu -i $out/r2c_cg.ncu-rep --page source --csv > $out/r2c_cg_source.csv 2>&1
rm -f $out/*.ncu-rep
cat $out/r2c_ab.txt
