out=gpurun_out; mkdir -p $out; rm -f $out/r2ab.txt
timeout 300 python scripts/ab_cg.py >> $out/r2ab.txt 2>&1
LBK_SOLVER_GRAPH=1 timeout 300 python scripts/ab_cg.py >> $out/r2ab.txt 2>&1
LBK_PDL=1 LBK_SOLVER_GRAPH=1 timeout 300 python scripts/ab_cg.py >> $out/r2ab.txt 2>&1
echo "== graph default" >> $out/r2ab.txt; timeout 300 python scripts/scale_probe.py 8 300 >> $out/r2ab.txt 2>&1
cat $out/r2ab.txt
