out=gpurun_out; mkdir -p $out; rm -f $out/r2ah.txt
timeout 300 python scripts/prof_pl.py >> $out/r2ah.txt 2>&1
timeout 300 python scripts/ab_spmv.py >> $out/r2ah.txt 2>&1
timeout 300 python scripts/ab_cg.py >> $out/r2ah.txt 2>&1
cat $out/r2ah.txt
