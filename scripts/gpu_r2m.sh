out=gpurun_out; mkdir -p $out
timeout 300 python scripts/ab_cg.py > $out/r2m.txt 2>&1
timeout 300 python scripts/phase_time.py >> $out/r2m.txt 2>&1
cat $out/r2m.txt
