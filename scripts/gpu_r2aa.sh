out=gpurun_out; mkdir -p $out; rm -f $out/r2aa.txt
for rep in 1 2 3; do
  echo "== pdl" >> $out/r2aa.txt; timeout 300 python scripts/scale_probe.py 8 300 >> $out/r2aa.txt 2>&1
  echo "== nopdl" >> $out/r2aa.txt; LBK_PDL=0 timeout 300 python scripts/scale_probe.py 8 300 >> $out/r2aa.txt 2>&1
done
timeout 300 python scripts/ab_cg.py >> $out/r2aa.txt 2>&1
LBK_PDL=0 timeout 300 python scripts/ab_cg.py >> $out/r2aa.txt 2>&1
cat $out/r2aa.txt
