out=gpurun_out; mkdir -p $out; rm -f $out/r2z.txt
for lib in default tree; do
  if [ $lib = tree ]; then export LBK_LIB=$PWD/_variants/liblbk_LBK_RED_TREE.so; fi
  echo "== $lib graph+pdl" >> $out/r2z.txt; timeout 300 python scripts/scale_probe.py 8 300 >> $out/r2z.txt 2>&1
  echo "== $lib nograph" >> $out/r2z.txt; LBK_SOLVER_GRAPH=0 timeout 300 python scripts/scale_probe.py 8 300 >> $out/r2z.txt 2>&1
  echo "== $lib nopdl" >> $out/r2z.txt; LBK_PDL=0 timeout 300 python scripts/scale_probe.py 8 300 >> $out/r2z.txt 2>&1
done
cat $out/r2z.txt
